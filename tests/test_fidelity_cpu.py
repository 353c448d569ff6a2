"""The fidelity harness (paper_2605_19660_b200/fidelity.py, mirroring
simulate_fidelity pipeline.cpp:359-408) driven by the CPU oracle: acceptance
criterion 7's method ordering (acceptance_main.cpp:278-335) must hold for the
harness itself before the device run is judged by it (tests/test_gpu_fidelity.py)."""
import numpy as np

from oracle import bindings as ob
from paper_2605_19660_b200 import fidelity as fd


class OracleCache:
    def __init__(self, method, bits, heads, max_tokens):
        self.c = ob.PortCache(method=method, bits=bits, H=heads)

    def append(self, k, v):
        self.c.append(k, v)

    def decode(self, q, k, v):
        return self.c.decode_step(q, k, v, 1)


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
    try:
        fd.preprocess(p)
        raise AssertionError("double preprocess must fail")
    except RuntimeError:
        pass


def test_method_ordering_with_oracle():
    cnt = fd.method_ordering(seeds=range(1, 7), cache_factory=OracleCache)
    assert cnt["oscar<rotate-only"] >= 5, cnt
    assert cnt["rotate-only<kivi"] >= 5, cnt
    assert cnt["scale-only>kivi"] >= 5, cnt
