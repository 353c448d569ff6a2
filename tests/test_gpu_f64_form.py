"""The reference's own call shapes on the device (kv_cache.hpp:80-84):
buffer_quant_k(K_u, norms) / buffer_quant_v(v) with fp64 rows that are NOT
bf16-representable (the reference's decode path feeds fp64 projections), the
decode step with the current token in that form, and KVC1 import of a cache the
reference built that way.  Packed codes, params, norms and the residual window
must equal the compiled reference's bit for bit; attention within the stated
tolerance (5e-3 * max|o|, as the raw path)."""
import os
import tempfile

import numpy as np
import pytest

from oracle import bindings as ob

from gpu_util import dev_bf16, export_to_oracle, log_err, rel_err

pytestmark = pytest.mark.gpu

TOL = 5e-3


def _keys(seed, S, H):
    """fp64 keys with the TNI outlier structure (offset / scaled channels, sink
    tokens) and fp64 values -- far from bf16-representable."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((S, H, 128)) * 0.7
    x[:, :, :4] += 18.0 * np.sign(rng.standard_normal((1, H, 4)))
    x[:, :, 4:12] *= 8.0
    x[:8] *= 0.01
    v = rng.standard_normal((S, H, 128))
    return x, v


def _dev64(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _need_ref():
    if not ob.ref_available():
        pytest.skip("oracle/_ref not built")


@pytest.mark.parametrize("bits,method,scaling", [(2, "oscar", "l2"), (4, "oscar", "rsqrt"), (2, "kivi", "l2"),
                                                 (2, "scale-only", "max")])
def test_buffer_quant_k_v_bit_exact(bits, method, scaling):
    """Prefill (S = 300: 2 blocks + 44 residual) then 150 single-token appends
    (a flush at 384) through buffer_quant_k / buffer_quant_v: the export equals the
    reference's KvCache fed the same rows, bit for bit, at every checkpoint."""
    _need_ref()
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    B, H, S, T = 2, 2, 300, 150
    cfg = PipelineConfig(method=method, bits=bits, scaling=scaling, heads=H)
    c = KvCache(cfg, batch=B, q_heads=H * 4, max_tokens=S + T + 8)
    xs, vs, kus, nrs = [], [], [], []
    for b in range(B):
        x, v = _keys(100 + b, S + T, H)
        ku, nr = ob.ref_apply_k(x, method, scaling)
        xs.append(x), vs.append(v), kus.append(ku), nrs.append(nr.reshape(S + T, H))
    refs = [ob.RefCache(method=method, bits=bits, scaling=scaling, H=H) for _ in range(B)]
    KU, NR, V = np.stack(kus), np.stack(nrs), np.stack(vs)
    c.buffer_quant_k(_dev64(KU[:, :S]), _dev64(NR[:, :S]))
    c.buffer_quant_v(_dev64(V[:, :S]))
    for b in range(B):
        refs[b].buffer_quant_k(kus[b][:S], nrs[b][:S])
        refs[b].buffer_quant_v(vs[b][:S])
    with tempfile.TemporaryDirectory() as td:
        for b in range(B):
            assert ob.caches_equal(export_to_oracle(c.export(b), H), refs[b].export(td)) == []
        for t in range(S, S + T):
            c.buffer_quant_k(_dev64(KU[:, t:t + 1]), _dev64(NR[:, t:t + 1]))
            c.buffer_quant_v(_dev64(V[:, t:t + 1]))
            for b in range(B):
                refs[b].buffer_quant_k(kus[b][t:t + 1], nrs[b][t:t + 1])
                refs[b].buffer_quant_v(vs[b][t:t + 1])
        assert (c.packed_tokens, c.residual_tokens, c.flush_count) == (384, 66, 1)
        for b in range(B):
            assert ob.caches_equal(export_to_oracle(c.export(b), H), refs[b].export(td)) == []
            # the device's own KVC1 dump of the fp64 form is the reference's dump, byte for byte
            pd, pr = os.path.join(td, "d.kvc1"), os.path.join(td, "r.kvc1")
            c.dump(b, pd)
            refs[b].dump(pr)
            assert open(pd, "rb").read() == open(pr, "rb").read()


def test_decode_step_f64_vs_reference():
    """decode_step with the current token as (K_u, norm, v) over 140 steps (a
    flush at step 84): outputs within tolerance of the reference's decode_step,
    and the cache bit-identical to the reference's afterwards."""
    _need_ref()
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    B, H, g, S, T = 2, 2, 4, 300, 140
    c = KvCache(PipelineConfig(heads=H, bits=2), batch=B, q_heads=H * g, max_tokens=S + T + 8)
    kus, nrs, vs, refs = [], [], [], []
    for b in range(B):
        x, v = _keys(200 + b, S + T, H)
        ku, nr = ob.ref_apply_k(x)
        kus.append(ku), nrs.append(nr.reshape(S + T, H)), vs.append(v)
        r = ob.RefCache(H=H)
        r.buffer_quant_k(ku[:S], nr[:S])
        r.buffer_quant_v(v[:S])
        refs.append(r)
    KU, NR, V = np.stack(kus), np.stack(nrs), np.stack(vs)
    c.buffer_quant_k(_dev64(KU[:, :S]), _dev64(NR[:, :S]))
    c.buffer_quant_v(_dev64(V[:, :S]))
    rng = np.random.default_rng(7)
    worst = 0.0
    for t in range(S, S + T):
        qf = rng.standard_normal((B, H * g, 128))
        q = dev_bf16(qf)
        qb = q.float().cpu().numpy().astype(np.float64)  # the bf16 q both sides attend with
        out = c.decode_step_f64(q, _dev64(KU[:, t]), _dev64(NR[:, t]), _dev64(V[:, t])).cpu().numpy()
        for b in range(B):
            want = refs[b].decode_step_f64(qb[b], kus[b][t], nrs[b][t], vs[b][t], g)
            worst = max(worst, rel_err(out[b].astype(np.float64), want))
    log_err("f64_form_decode_140_steps", worst)
    assert worst <= TOL, worst
    assert (c.packed_tokens, c.residual_tokens, c.flush_count) == (384, 56, 1)
    with tempfile.TemporaryDirectory() as td:
        for b in range(B):
            assert ob.caches_equal(export_to_oracle(c.export(b), H), refs[b].export(td)) == []


def test_reference_fp64_cache_loads_on_device():
    """A KVC1 file the reference wrote for a cache built from fp64 rows (the
    residual rows are not bf16 transforms) loads on the device in the fp64 form:
    export equals the reference's, re-dump is byte-identical, and decoding
    continues like the reference."""
    _need_ref()
    from paper_2605_19660_b200 import KvCache, PipelineConfig
    from paper_2605_19660_b200.kv_cache import read_kvc1_config

    H, g, S = 2, 4, 330
    x, v = _keys(300, S + 3, H)
    ku, nr = ob.ref_apply_k(x)
    nr = nr.reshape(S + 3, H)
    ref = ob.RefCache(H=H)
    ref.buffer_quant_k(ku[:S], nr[:S])
    ref.buffer_quant_v(v[:S])
    with tempfile.TemporaryDirectory() as td:
        p, p2 = os.path.join(td, "ref.kvc1"), os.path.join(td, "dev.kvc1")
        ref.dump(p)
        cfg, tokens = read_kvc1_config(p)
        assert (cfg.bits, cfg.heads, cfg.method, tokens) == (2, H, "oscar", S)
        c = KvCache(cfg, batch=1, q_heads=H * g, max_tokens=S + 8)
        c.load(0, p)
        assert ob.caches_equal(export_to_oracle(c.export(0), H), ref.export(td)) == []
        c.dump(0, p2)
        assert open(p, "rb").read() == open(p2, "rb").read()
    rng = np.random.default_rng(9)
    for t in range(S, S + 3):
        q = dev_bf16(rng.standard_normal((1, H * g, 128)))
        qb = q.float().cpu().numpy().astype(np.float64)[0]
        got = c.decode_step_f64(q, _dev64(ku[None, t]), _dev64(nr[None, t]), _dev64(v[None, t])).cpu().numpy()[0]
        want = ref.decode_step_f64(qb, ku[t], nr[t], v[t], g)
        assert rel_err(got.astype(np.float64), want) <= TOL


def test_streams_and_forms():
    """K and V advance separately like the reference's k_/v_ state; attention
    needs them in step; one input form per cache; config restrictions."""
    import torch

    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H = 1
    c = KvCache(PipelineConfig(heads=H, bits=2), batch=1, q_heads=4, max_tokens=512)
    x, v = _keys(5, 140, H)
    nr = np.linalg.norm(x, axis=2)  # any fp64 rows are valid input; the form is what is tested
    ku = x / nr[:, :, None]
    c.buffer_quant_k(_dev64(ku[None, :130]), _dev64(nr[None, :130]))
    assert (c.packed_tokens, c.residual_tokens) == (128, 2)
    assert c.v_tokens == (0, 0)
    q = dev_bf16(np.ones((1, 4, 128)))
    with pytest.raises(RuntimeError):  # status 2: streams out of step
        c.attend(q)
    c.buffer_quant_v(_dev64(v[None, :130]))
    assert c.v_tokens == (128, 2)
    c.attend(q)
    with pytest.raises(RuntimeError):  # raw bf16 appends cannot join an fp64-form cache
        c.buffer_quant(dev_bf16(x[None, :1]), dev_bf16(v[None, :1]))
    raw = KvCache(PipelineConfig(heads=H, bits=2), batch=1, q_heads=4, max_tokens=512)
    raw.buffer_quant(dev_bf16(x[None, :10]), dev_bf16(v[None, :10]))
    with pytest.raises(RuntimeError):
        raw.buffer_quant_k(_dev64(ku[None, :1]), _dev64(nr[None, :1]))
    for cfg in (PipelineConfig(heads=H, bits=0), PipelineConfig(heads=H, bits=2, rotate_v=True)):
        bad = KvCache(cfg, batch=1, q_heads=4, max_tokens=512)
        with pytest.raises(ValueError):
            bad.buffer_quant_k(_dev64(ku[None, :1]), _dev64(nr[None, :1]))
    with pytest.raises(ValueError):  # fp32 rows are not the reference's form
        c.buffer_quant_v(torch.zeros((1, 1, H, 128), dtype=torch.float32, device="cuda"))
