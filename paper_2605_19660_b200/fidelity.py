"""Fidelity harness on the device path, mirroring the reference's
simulate_fidelity (pipeline.cpp:359-408) and acceptance criterion 7
(acceptance_main.cpp:278-335): a single-layer model stub projects hidden
states to q/k/v, a prompt is prefilled into the cache, then every decode row
runs decode_step and the attention output (through W_O) and the attention
logits (StepOutput.logits) are compared with the unquantised ("fp") path.
Only the cache path is ours; the projections are fp64 numpy matmuls
(plumbing, outside the path) whose results are rounded
to bf16, the device cache's input type.

The hidden rows and stub weights can come from anywhere; the parity tests
feed the ones the REFERENCE generates for criterion 7 (generate(TniSpec) and
make_sim_stub with its SeededRng, through oracle/_ref) and compare the
device's output / logit MSEs with the reference's own simulate_fidelity on
the same rows.

The method variants (kivi, rotate-only, scale-only, oscar) are flags of the
same kernels.  For oscar the weights are folded first (preprocess,
pipeline.cpp:38-78): W_V <- W_V (I (x) Hn), W_O <- (I (x) Hn) W_O, so the
cache stores rotated V exactly as the reference's cache does.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .synthetic import round_bf16


@dataclass
class ModelStub:
    """make_sim_stub (pipeline.cpp:327-357): W_K = I, W_Q = diag(+-gain),
    W_V block-diagonal per head (value_mix * I + (1 - value_mix) N(0,1)/sqrt(d)),
    W_O dense N(0,1)/sqrt(d_model)."""

    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray
    heads: int
    head_dim: int
    preprocessed: bool = False


def make_sim_stub(heads: int, head_dim: int, rng: np.random.Generator, query_gain: float = 0.12,
                  value_mix: float = 0.5) -> ModelStub:
    dm = heads * head_dim
    w_q = np.diag(np.where(rng.random(dm) < 0.5, -query_gain, query_gain))
    w_v = np.zeros((dm, dm))
    hs = 1.0 / np.sqrt(head_dim)
    for h in range(heads):
        blk = (1.0 - value_mix) * rng.standard_normal((head_dim, head_dim)) * hs + value_mix * np.eye(head_dim)
        w_v[h * head_dim:(h + 1) * head_dim, h * head_dim:(h + 1) * head_dim] = blk
    w_o = rng.standard_normal((dm, dm)) / np.sqrt(dm)
    return ModelStub(w_q, np.eye(dm), w_v, w_o, heads, head_dim)


def hadamard_matrix(d: int) -> np.ndarray:
    """Normalized Sylvester Hadamard matrix (hadamard.cpp:45-64)."""
    if d & (d - 1):
        raise ValueError("hadamard_matrix: d must be a power of two")
    h = np.array([[1.0]])
    while h.shape[0] < d:
        h = np.block([[h, h], [h, -h]])
    return h / np.sqrt(d)


def preprocess(model: ModelStub) -> ModelStub:
    """preprocess (pipeline.cpp:38-78): fold Hn into W_V columns and W_O rows."""
    if model.preprocessed:
        raise RuntimeError("preprocess: model is already preprocessed")  # logic_error
    f = np.kron(np.eye(model.heads), hadamard_matrix(model.head_dim))
    return ModelStub(model.w_q, model.w_k, model.w_v @ f, f @ model.w_o, model.heads, model.head_dim, True)


class DeviceCache:
    """Adapter: numpy bf16-valued [T, H, d] in, fp32 attention rows + logits
    out, over the device KvCache (one sequence, MHA as in the reference)."""

    def __init__(self, method: str, bits: int, heads: int, max_tokens: int, device: int = 0,
                 scaling: str = "l2"):
        from .kv_cache import KvCache, PipelineConfig

        self.cache = KvCache(PipelineConfig(method=method, bits=bits, heads=heads, scaling=scaling), batch=1,
                             q_heads=heads, max_tokens=max_tokens, device=device, keep_exact=False)
        self.device = device

    def _dev(self, x):
        import torch

        return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(f"cuda:{self.device}").to(torch.bfloat16)

    def append(self, k, v):
        self.cache.buffer_quant(self._dev(k)[None], self._dev(v)[None])

    def decode(self, q, k, v):
        """-> (attention rows [H, d], logits [H, S_total]) of one decode step."""
        import torch

        lg = torch.empty((1, q.shape[0], self.cache.total_tokens + 1), dtype=torch.float32,
                         device=f"cuda:{self.device}")
        out = self.cache.decode_step(self._dev(q)[None], self._dev(k)[None], self._dev(v)[None], logits=lg)
        return out[0].double().cpu().numpy(), lg[0].double().cpu().numpy()

    @property
    def flush_count(self):
        return self.cache.flush_count

    def memory_report(self):
        return self.cache.memory_report()

    def close(self):
        self.cache.close()


@dataclass
class FidelityReport:
    """FidelityReport (pipeline.hpp:87-94).  prefill_output_mse is None: the
    prefill attention (attention_causal over the un-quantised current tensors,
    pipeline.cpp:262-268) is not part of the device path."""

    output_mse: float
    logit_mse: float
    flushes: int
    decode_steps: int
    memory: dict = None
    prefill_output_mse: float = None


def simulate_fidelity(model: ModelStub, hidden: np.ndarray, prefill: int, method: str, bits: int = 2,
                      scaling: str = "l2", cache_factory=None) -> FidelityReport:
    """simulate_fidelity (pipeline.cpp:359-408) for one method: output and
    logit MSE of the decode rows against the fp path (method "fp", the exact
    bf16 cache).  hidden: [T, heads*head_dim]; rows [0, prefill) are the
    prompt, the rest are decode rows.  For oscar the folded weights are used
    (preprocess), exactly as the reference does."""
    factory = cache_factory or (lambda m, b, h, n, sc: DeviceCache(m, b, h, n, scaling=sc))
    H, d = model.heads, model.head_dim
    T = hidden.shape[0]
    outs, logits, caches = {}, {}, {}
    for m in ("fp", method):
        run = preprocess(model) if m == "oscar" else model
        q = round_bf16(hidden @ run.w_q).reshape(T, H, d)
        k = round_bf16(hidden @ run.w_k).reshape(T, H, d)
        v = round_bf16(hidden @ run.w_v).reshape(T, H, d)
        cache = factory(m, 0 if m == "fp" else bits, H, T + 8, scaling)
        cache.append(k[:prefill], v[:prefill])
        rows, lgs = [], []
        for t in range(prefill, T):
            o, lg = cache.decode(q[t], k[t], v[t])
            rows.append(o.reshape(-1) @ run.w_o)
            lgs.append(lg.reshape(-1))
        outs[m] = np.array(rows)
        logits[m] = lgs
        caches[m] = cache
    mse = float(np.mean((outs[method] - outs["fp"]) ** 2))
    lmse = float(np.mean(np.concatenate([(a - b) ** 2 for a, b in zip(logits[method], logits["fp"])])))
    c = caches[method]
    rep = FidelityReport(mse, lmse, int(getattr(c, "flush_count", 0)), T - prefill,
                         c.memory_report() if hasattr(c, "memory_report") else None)
    for cc in caches.values():
        if hasattr(cc, "close"):
            cc.close()
    return rep


def method_ordering(inputs, cache_factory=None) -> dict:
    """Acceptance criterion 7 (acceptance_main.cpp:278-335): counts of
    oscar < rotate-only, rotate-only < kivi and scale-only > kivi over the
    given (hidden, model, prefill) inputs (the reference requires >= 18 of
    20 each); also returns every output MSE."""
    cnt = {"oscar<rotate-only": 0, "rotate-only<kivi": 0, "scale-only>kivi": 0, "seeds": 0, "mse": []}
    for hidden, model, prefill in inputs:
        mse = {m: simulate_fidelity(model, hidden, prefill, m, cache_factory=cache_factory).output_mse
               for m in ("kivi", "rotate-only", "scale-only", "oscar")}
        cnt["oscar<rotate-only"] += mse["oscar"] < mse["rotate-only"]
        cnt["rotate-only<kivi"] += mse["rotate-only"] < mse["kivi"]
        cnt["scale-only>kivi"] += mse["scale-only"] > mse["kivi"]
        cnt["seeds"] += 1
        cnt["mse"].append(mse)
    return cnt


def synthetic_inputs(seeds=range(1, 21), prefill: int = 256, decode: int = 64, heads: int = 4,
                     head_dim: int = 128):
    """numpy stand-ins for criterion 7's inputs (TNI hidden rows + stub), for
    runs without the compiled reference."""
    from .synthetic import tni_keys

    for seed in seeds:
        rng = np.random.default_rng(seed)
        hidden = tni_keys(rng, prefill + decode, heads, head_dim).reshape(prefill + decode, heads * head_dim)
        yield hidden, make_sim_stub(heads, head_dim, rng), prefill
