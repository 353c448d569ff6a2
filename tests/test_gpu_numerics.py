"""The decode kernel's deviation from the fp64 oracle is its fp16 operand
roundings (tests/fp16_model.py): the GPU output sits much closer to the
rounding model than to the oracle, and the model with roundings off IS the
oracle (tests/test_fp16_model_cpu.py).

Keys with DC outlier channels (the test_gpu_scale.py distribution) give a
logit spread of ~5-6 log2 units per sigma, where the ~2^-12 operand roundings
reach a few 1e-3 of max|out|; the model pins where that error comes from.
"""
import numpy as np
import pytest

from oracle import bindings as ob

from fp16_model import emulate, head_arrays
from gpu_util import dev_bf16, export_to_oracle, log_err, rel_err

pytestmark = pytest.mark.gpu


def _bf16(x):
    from paper_2605_19660_b200.synthetic import to_bf16_bits

    u = to_bf16_bits(np.ascontiguousarray(x, np.float32)).astype(np.uint32) << 16
    return u.view(np.float32).astype(np.float64)


@pytest.mark.parametrize("bits", [2, 4])
def test_kernel_equals_fp16_rounding_model(bits):
    import torch

    from paper_2605_19660_b200 import KvCache, PipelineConfig

    rng = np.random.default_rng(40 + bits)
    S, H, g, d = 8192, 2, 4, 128
    k = rng.standard_normal((1, S, H, d))
    k[..., 0:4] = 18.0 * np.sign(rng.standard_normal((1, 1, H, 4))) + 0.3 * k[..., 0:4]
    k[..., 4:12] *= 8.0
    v = rng.standard_normal((1, S, H, d))
    q = rng.standard_normal((1, H * g, d))
    k, v, q = _bf16(k), _bf16(v), _bf16(q)

    cache = KvCache(PipelineConfig(heads=H, bits=bits), batch=1, q_heads=H * g, max_tokens=S + 8)
    cache.buffer_quant(dev_bf16(k), dev_bf16(v))
    assert cache.residual_tokens == 0
    out, _ = cache.attend(dev_bf16(q))
    out = out.float().cpu().numpy().astype(np.float64)[0]
    torch.cuda.synchronize()

    ec = export_to_oracle(cache.export(0), H)
    worst_model, worst_oracle = 0.0, 0.0
    for h in range(H):
        K, V, norms = head_arrays(ec, h)
        for j in range(g):
            row = h * g + j
            qr = ob.port_fht(q[0, row])
            model = emulate(qr, K, V, norms)
            exact = emulate(qr, K, V, norms, on=())
            worst_model = max(worst_model, rel_err(out[row], model))
            worst_oracle = max(worst_oracle, rel_err(out[row], exact))
    log_err(f"fp16_model[bits={bits}][S={S},H={H},g={g}] vs model", worst_model)
    log_err(f"fp16_model[bits={bits}][S={S},H={H},g={g}] vs oracle", worst_oracle)
    # The model reproduces the key-side roundings exactly (q16, a16, b16, q16*a16
    # are data-determined); the value-side P and P*a roundings happen relative to
    # each warp's running max, which the model replaces by the global max, so
    # those ~5e-4 draws differ: the kernel sits within that of the model and
    # well inside the oracle tolerance.
    assert worst_model <= 1.2e-3, worst_model
    assert worst_model < 0.5 * worst_oracle, (worst_model, worst_oracle)
    assert worst_oracle <= 1e-2, worst_oracle


@pytest.mark.parametrize("bits", [2, 4])
def test_large_value_magnitudes_stay_finite(bits):
    """Values of magnitude ~2000 (group ranges ~9000): the fp16 steps and the
    P*a fold (P <= 2^3 between lazy rescales) stay finite; the output matches
    the oracle within the attention tolerance."""
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    rng = np.random.default_rng(70 + bits)
    S, H, g, d = 2048, 2, 4, 128
    k = _bf16(rng.standard_normal((1, S + 1, H, d)) * 3.0)
    v = _bf16(rng.standard_normal((1, S + 1, H, d)) * 2000.0)
    q = _bf16(rng.standard_normal((1, H * g, d)))
    cache = KvCache(PipelineConfig(heads=H, bits=bits), batch=1, q_heads=H * g, max_tokens=S + 8)
    cache.buffer_quant(dev_bf16(k[:, :S]), dev_bf16(v[:, :S]))
    out = cache.decode_step(dev_bf16(q), dev_bf16(k[:, S]), dev_bf16(v[:, S])).cpu().numpy()[0].astype(np.float64)
    assert np.isfinite(out).all()
    o = ob.PortCache(H=H, bits=bits)
    o.append(k[0, :S], v[0, :S])
    ref = o.decode_step(q[0], k[0, S], v[0, S], g, append=False)
    err = rel_err(out, ref)
    log_err(f"large_values[bits={bits}][|v|~2000]", err)
    assert err <= 5e-3, err


def test_device_status_flags():
    """oscar_kv_status: finite inputs in range raise nothing; a value range beyond
    the fp16 step/offset raises FP16_OVERFLOW (the exported fp64 params stay
    bit-exact with the oracle); a non-finite input raises NONFINITE; clear resets."""
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    rng = np.random.default_rng(5)
    S, H, d = 256, 2, 128
    k = _bf16(rng.standard_normal((1, S, H, d)))
    v = _bf16(rng.standard_normal((1, S, H, d)))
    c = KvCache(PipelineConfig(heads=H, bits=2), batch=1, q_heads=H * 4, max_tokens=S + 8)
    c.buffer_quant(dev_bf16(k), dev_bf16(v))
    assert c.status()["raw"] == 0

    big = v.copy()
    big[0, 5, 1, :] *= 1e6  # one token's value groups span ~1e6: the fp16 step overflows
    big = _bf16(big)
    c2 = KvCache(PipelineConfig(heads=H, bits=2), batch=1, q_heads=H * 4, max_tokens=S + 8)
    c2.buffer_quant(dev_bf16(k), dev_bf16(big))
    st = c2.status()
    assert st["fp16_overflow"] and not st["nonfinite_input"], st
    o = ob.PortCache(H=H, bits=2)
    o.append(k[0], big[0])
    assert ob.caches_equal(export_to_oracle(c2.export(0), H), o.export()) == []
    assert c2.status(clear=True)["raw"] != 0 and c2.status()["raw"] == 0

    bad = k.copy()
    bad[0, 7, 0, 3] = np.nan
    c3 = KvCache(PipelineConfig(heads=H, bits=2), batch=1, q_heads=H * 4, max_tokens=S + 8)
    c3.buffer_quant(dev_bf16(bad), dev_bf16(v))
    assert c3.status()["nonfinite_input"]
