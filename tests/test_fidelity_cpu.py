"""The fidelity harness (paper_2605_19660_b200/fidelity.py, mirroring
simulate_fidelity pipeline.cpp:359-408) driven on the CPU, before the device
run is judged by it (tests/test_gpu_fidelity.py):

* its inputs are the reference's own: generate(TniSpec) hidden rows and the
  make_sim_stub weights of acceptance criterion 7 (acceptance_main.cpp:
  282-312), produced by the compiled reference (oracle/_ref);
* driven through the compiled reference's KvCache + attention (RefCache) on
  the bf16-rounded projections the device sees, its output / logit MSEs track
  the reference's simulate_fidelity on the fp64 rows, and criterion 7's
  orderings hold;
* our numpy preprocess equals the reference's preprocess."""
import numpy as np
import pytest

from oracle import bindings as ob
from paper_2605_19660_b200 import fidelity as fd

needs_ref = pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built")


class RefHarnessCache:
    """fidelity.py cache adapter over the compiled reference (RefCache)."""

    def __init__(self, method, bits, heads, max_tokens, scaling="l2"):
        self.c = ob.RefCache(method=method, bits=bits, H=heads, scaling=scaling)

    def append(self, k, v):
        self.c.append(k, v)

    def decode(self, q, k, v):
        return self.c.decode_step_logits(q, k, v, 1)

    @property
    def flush_count(self):
        return self.c.stats()["flushes"]

    def memory_report(self):
        return self.c.memory_report()


def model_from_ref(seed, S=256, Dn=64):
    hidden, (wq, wk, wv, wo) = ob.ref_crit7_inputs(seed, S, Dn)
    return hidden, fd.ModelStub(wq, wk, wv, wo, 4, 128), S


def test_stub_and_preprocess_shapes():
    rng = np.random.default_rng(3)
    m = fd.make_sim_stub(2, 128, rng)
    assert m.w_q.shape == (256, 256) and np.allclose(np.abs(np.diag(m.w_q)), 0.12)
    assert np.count_nonzero(m.w_v[:128, 128:]) == 0  # block-diagonal per head
    p = fd.preprocess(m)
    h = fd.hadamard_matrix(128)
    assert np.allclose(h @ h, np.eye(128))  # self-inverse (test_hadamard.cpp:29-77)
    # folding preserves the layer: W_V' W_O' == W_V W_O (pipeline.cpp:38-78)
    assert np.allclose(p.w_v @ p.w_o, m.w_v @ m.w_o)
    with pytest.raises(RuntimeError):
        fd.preprocess(p)


@needs_ref
def test_preprocess_matches_reference():
    hidden, m, _ = model_from_ref(3)
    wv, wo = ob.ref_preprocess(m.w_v, m.w_o)
    p = fd.preprocess(m)
    assert np.max(np.abs(p.w_v - wv)) <= 1e-12 * np.max(np.abs(wv))
    assert np.max(np.abs(p.w_o - wo)) <= 1e-12 * np.max(np.abs(wo))


@needs_ref
def test_harness_tracks_reference_simulate_fidelity():
    """Same rows, same weights: the harness (bf16-rounded projections into the
    reference's own cache) vs the reference's simulate_fidelity (fp64 rows).
    The bf16 input rounding is small next to the 2-bit quantisation error."""
    ob.ref_use_threads(8)
    for seed in (1, 2):
        hidden, m, S = model_from_ref(seed)
        for method in ("kivi", "oscar"):
            mine = fd.simulate_fidelity(m, hidden, S, method, cache_factory=RefHarnessCache)
            ref = ob.ref_simulate_fidelity(hidden, S, [m.w_q, m.w_k, m.w_v, m.w_o], method)
            assert 0.85 < mine.output_mse / ref["output_mse"] < 1.15, (seed, method, mine, ref)
            assert 0.85 < mine.logit_mse / ref["logit_mse"] < 1.15, (seed, method, mine, ref)
            assert mine.flushes == ref["flushes"] and mine.decode_steps == ref["decode_steps"]
            assert mine.memory == ref["memory"]


@needs_ref
def test_method_ordering_with_reference_cache():
    ob.ref_use_threads(8)
    cnt = fd.method_ordering([model_from_ref(s) for s in range(1, 7)], cache_factory=RefHarnessCache)
    assert cnt["oscar<rotate-only"] >= 5, cnt
    assert cnt["rotate-only<kivi"] >= 5, cnt
    assert cnt["scale-only>kivi"] >= 5, cnt
