"""Pins tests/fp16_model.py: with its roundings off it IS the oracle's attention
(pipeline.cpp:152-180) over the materialized cache, so the GPU test
test_gpu_numerics.py can attribute the kernel's deviation to the roundings."""
import numpy as np

from oracle import bindings as ob

from fp16_model import emulate, f16, head_arrays


def test_model_without_roundings_is_the_oracle():
    rng = np.random.default_rng(7)
    S, H, d = 1024, 1, 128
    k = f16(rng.standard_normal((S, H, d)) * 3.0)
    v = f16(rng.standard_normal((S, H, d)))
    o = ob.PortCache(H=H, bits=4)
    o.append(k, v)
    K, V, norms = head_arrays(o.export(), 0)
    qr = ob.port_fht(f16(rng.standard_normal(d)))
    km, vm = o.materialize()  # rotated-space keys x norm (kv_cache.cpp:327-381)
    logits = km[:, 0] @ qr / np.sqrt(d)
    w = np.exp(logits - logits.max())
    ref = (w[:, None] * vm[:, 0]).sum(0) / w.sum()
    exact = emulate(qr, K, V, norms, on=())
    assert np.max(np.abs(exact - ref)) <= 1e-12 * np.max(np.abs(ref))
    # and the roundings do move it, by a few 2^-12
    assert 0 < np.max(np.abs(emulate(qr, K, V, norms) - ref)) <= 1e-2 * np.max(np.abs(ref))
