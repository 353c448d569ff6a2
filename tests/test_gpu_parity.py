"""Parity of the CUDA path (through the C-ABI) against the CPU oracle.

Bar:
  * quantize/append: codes, delta, zero point, constant, norms and the
    residual window BIT-EXACT against oracle/oscar_oracle.c (itself pinned to
    the compiled reference) and the KVC1 dump BYTE-identical to the
    reference's own dump when oracle/_ref is present;
  * decode attention: fp32 output within ATOL_REL * max|o| of the fp64
    oracle (q/K/V enter as bf16; the kernel folds steps into fp16 operands and
    accumulates in fp32) -- the tolerance is stated below.
"""
import os
import tempfile

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2605_19660_b200.synthetic import make_inputs, make_queries

from gpu_util import dev_bf16, export_to_oracle, log_err, rel_err

pytestmark = pytest.mark.gpu

# attention tolerance: max |o_dev - o_oracle| <= ATOL_REL * max |o_oracle|
ATOL_REL_QUANT = 5e-3   # packed INT2/INT4 path (fp16 folded steps, fp16 P): <= 2.5 bf16 half-ulps
ATOL_REL_BF16 = 1e-2    # bf16 exact-cache baseline (bf16 P)

CONFIGS = [
    # method, bits, scaling, rotate_v, H, g
    ("oscar", 2, "l2", False, 2, 4),
    ("oscar", 2, "rsqrt", False, 2, 4),
    ("oscar", 2, "max", False, 1, 7),
    ("oscar", 2, "mean-abs", False, 2, 4),
    ("oscar", 4, "l2", False, 2, 4),
    ("oscar", 2, "l2", True, 2, 4),
    ("kivi", 2, "l2", False, 2, 4),
    ("kivi", 4, "l2", False, 1, 8),
    ("rotate-only", 2, "l2", False, 2, 4),
    ("scale-only", 2, "l2", False, 2, 1),
    ("oscar", 0, "l2", False, 2, 4),
    ("fp", 2, "l2", False, 2, 4),
]


def _ids(c):
    return "-".join(map(str, c))


def _build(cfg_t, B, S_pre, S_app, seed):
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    method, bits, scaling, rotv, H, g = cfg_t
    cfg = PipelineConfig(method=method, bits=bits, scaling=scaling, heads=H, rotate_v=rotv)
    S = S_pre + S_app
    data = [make_inputs(seed + b, S + 1, H) for b in range(B)]
    cache = KvCache(cfg, batch=B, q_heads=H * g, max_tokens=S + 64)
    cache.buffer_quant(dev_bf16(np.stack([d[0][:S_pre] for d in data])),
                       dev_bf16(np.stack([d[1][:S_pre] for d in data])))
    for t in range(S_pre, S):
        cache.buffer_quant(dev_bf16(np.stack([d[0][t : t + 1] for d in data])),
                           dev_bf16(np.stack([d[1][t : t + 1] for d in data])))
    oracles = []
    for b in range(B):
        o = ob.PortCache(method=method, bits=bits, scaling=scaling, H=H, rotate_v=rotv)
        o.append(data[b][0][:S_pre], data[b][1][:S_pre])
        for t in range(S_pre, S):
            o.append(data[b][0][t : t + 1], data[b][1][t : t + 1])
        oracles.append(o)
    return cache, oracles, data


@pytest.mark.parametrize("cfg_t", CONFIGS, ids=_ids)
def test_quantize_append_bitexact(cfg_t):
    # prefill 250 (1 packed block + 122 residual) then 10 single-token appends:
    # the 6th append flushes the window at exactly R (kv_cache.cpp:228-248)
    cache, oracles, _ = _build(cfg_t, B=2, S_pre=250, S_app=10, seed=1000)
    assert (cache.packed_tokens, cache.residual_tokens, cache.flush_count) == (256, 4, 1)
    for b, o in enumerate(oracles):
        mine = export_to_oracle(cache.export(b), cfg_t[4])
        assert ob.caches_equal(mine, o.export()) == []
        km, vm = cache.materialize(b)
        ko, vo = o.materialize()
        assert np.array_equal(km, ko) and np.array_equal(vm, vo)


@pytest.mark.parametrize("cfg_t", CONFIGS, ids=_ids)
def test_decode_step_matches_oracle(cfg_t):
    method, bits, scaling, rotv, H, g = cfg_t
    B = 3
    cache, oracles, data = _build(cfg_t, B=B, S_pre=300, S_app=0, seed=2000)
    q = np.stack([make_queries(2000 + b, 1, H * g)[0] for b in range(B)])
    out = cache.decode_step(dev_bf16(q), dev_bf16(np.stack([d[0][300] for d in data])),
                            dev_bf16(np.stack([d[1][300] for d in data]))).cpu().numpy()
    tol = ATOL_REL_QUANT if (bits and method != "fp") else ATOL_REL_BF16
    for b, o in enumerate(oracles):
        ref = o.decode_step(q[b], data[b][0][300], data[b][1][300], g)
        if rotv:
            ref = np.stack([ob.port_fht(r) for r in ref])
        err = rel_err(out[b].astype(np.float64), ref)
        log_err(f"decode_step[{_ids(cfg_t)}][b={b}]", err)
        assert err <= tol, (b, err)
    # the current token landed in the residual window, after the attention
    assert cache.total_tokens == 301 and cache.residual_tokens == 301 - 256


def test_flush_consistency_on_device():
    """prefill(S) == empty prefill + S single-token appends (test_kv_cache.cpp:137-176)."""
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H, S = 2, 300
    k, v = make_inputs(41, S, H)
    cfg = PipelineConfig(heads=H)
    a = KvCache(cfg, batch=1, q_heads=H, max_tokens=512)
    a.buffer_quant(dev_bf16(k[None]), dev_bf16(v[None]))
    b = KvCache(cfg, batch=1, q_heads=H, max_tokens=512)
    b.buffer_quant(dev_bf16(k[None, :0]), dev_bf16(v[None, :0]))
    for t in range(S):
        b.buffer_quant(dev_bf16(k[None, t : t + 1]), dev_bf16(v[None, t : t + 1]))
    ea, eb = export_to_oracle(a.export(0), H), export_to_oracle(b.export(0), H)
    eb.flush_count = ea.flush_count  # the stepped cache counts its decode-branch flushes
    assert ob.caches_equal(ea, eb) == []


def test_decode_loop_crosses_flushes():
    """140 decode steps from S=120: flush at R inside the loop, outputs track the oracle."""
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H, g, S0, steps = 2, 4, 120, 140
    k, v = make_inputs(7, S0 + steps, H)
    q = make_queries(7, steps, H * g)
    cache = KvCache(PipelineConfig(heads=H), batch=1, q_heads=H * g, max_tokens=512)
    cache.buffer_quant(dev_bf16(k[None, :S0]), dev_bf16(v[None, :S0]))
    o = ob.PortCache(H=H)
    o.append(k[:S0], v[:S0])
    worst = 0.0
    for i in range(steps):
        t = S0 + i
        out = cache.decode_step(dev_bf16(q[i][None]), dev_bf16(k[t][None]), dev_bf16(v[t][None])).cpu().numpy()
        ref = o.decode_step(q[i], k[t], v[t], g)
        worst = max(worst, rel_err(out[0].astype(np.float64), ref))
    log_err("decode_loop_140_steps(worst)", worst)
    assert worst <= ATOL_REL_QUANT, worst
    assert (cache.packed_tokens, cache.residual_tokens, cache.flush_count) == (256, 4, 2)
    assert ob.caches_equal(export_to_oracle(cache.export(0), H), o.export()) == []


def test_first_decode_after_empty_prefill_attends_itself():
    # test_pipeline.cpp:231-245: softmax over one token -> output = v
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H, g = 2, 4
    k, v = make_inputs(3, 1, H)
    q = make_queries(3, 1, H * g)
    cache = KvCache(PipelineConfig(heads=H), batch=1, q_heads=H * g, max_tokens=64)
    cache.buffer_quant(dev_bf16(k[None, :0]), dev_bf16(v[None, :0]))
    out = cache.decode_step(dev_bf16(q), dev_bf16(k[0][None]), dev_bf16(v[0][None])).cpu().numpy()
    for h in range(H * g):
        assert np.allclose(out[0, h], v[0, h // g], atol=1e-6)


def test_prefill_multiple_of_R_and_short_prefill():
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H = 2
    for S, packed, res in ((256, 256, 0), (100, 0, 100), (129, 128, 1)):
        k, v = make_inputs(S, S, H)
        c = KvCache(PipelineConfig(heads=H), batch=2, q_heads=H, max_tokens=512)
        c.buffer_quant(dev_bf16(np.stack([k, k])), dev_bf16(np.stack([v, v])))
        assert (c.packed_tokens, c.residual_tokens) == (packed, res)
        o = ob.PortCache(H=H)
        o.append(k, v)
        assert ob.caches_equal(export_to_oracle(c.export(1), H), o.export()) == []


def test_errors_map_to_reference_exception_types():
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    with pytest.raises(ValueError):
        PipelineConfig(residual_len=100).validate()
    with pytest.raises(ValueError):
        PipelineConfig(bits=5).validate()
    with pytest.raises(ValueError):
        KvCache(PipelineConfig(heads=2), batch=1, q_heads=3, max_tokens=10)
    c = KvCache(PipelineConfig(heads=1), batch=1, q_heads=1, max_tokens=10)
    k, v = make_inputs(1, 20, 1)
    with pytest.raises(ValueError):
        c.buffer_quant(dev_bf16(k[None]), dev_bf16(v[None]))


def test_dump_is_byte_identical_to_reference_dump():
    if not ob.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    for bits in (2, 4, 0):
        H, S = 2, 300
        k, v = make_inputs(50 + bits, S, H)
        c = KvCache(PipelineConfig(heads=H, bits=bits), batch=1, q_heads=H, max_tokens=512)
        c.buffer_quant(dev_bf16(k[None, :290]), dev_bf16(v[None, :290]))
        for t in range(290, S):
            c.buffer_quant(dev_bf16(k[None, t : t + 1]), dev_bf16(v[None, t : t + 1]))
        ref = ob.RefCache(H=H, bits=bits)
        ref.append(k[:290], v[:290])
        for t in range(290, S):
            ref.append(k[t : t + 1], v[t : t + 1])
        with tempfile.TemporaryDirectory() as td:
            pa, pb = os.path.join(td, "dev.kvc1"), os.path.join(td, "ref.kvc1")
            c.dump(0, pa)
            ref.dump(pb)
            assert open(pa, "rb").read() == open(pb, "rb").read(), bits
            # and the reference loads our dump back
            back = ob.RefCache.load(pa, H=H, d=128)
            assert back.stats() == ref.stats()


def test_host_buffer_entry_matches_device_entry():
    from paper_2605_19660_b200 import KvCache, PipelineConfig
    from paper_2605_19660_b200.synthetic import to_bf16_bits

    H, g, S = 2, 4, 200
    k, v = make_inputs(9, S + 1, H)
    q = make_queries(9, 1, H * g)
    import torch

    outs, lses = [], []
    # device entry; host entry with pageable buffers (D2H copies); host entry with
    # page-locked buffers (the kernel writes out/lse to mapped host memory)
    for mode in ("device", "pageable", "pinned"):
        c = KvCache(PipelineConfig(heads=H), batch=1, q_heads=H * g, max_tokens=512)
        c.buffer_quant(dev_bf16(k[None, :S]), dev_bf16(v[None, :S]))
        if mode == "device":
            lse = torch.empty((1, H * g), device="cuda")
            outs.append(c.decode_step(dev_bf16(q), dev_bf16(k[S][None]), dev_bf16(v[S][None]), lse=lse).cpu().numpy())
            lses.append(lse.cpu().numpy())
            continue
        qb, kb, vb = to_bf16_bits(q), to_bf16_bits(k[S][None]), to_bf16_bits(v[S][None])
        if mode == "pageable":
            o, l = np.zeros((1, H * g, 128), np.float32), np.zeros((1, H * g), np.float32)
        else:
            ot = torch.zeros((1, H * g, 128), dtype=torch.float32).pin_memory()
            lt = torch.zeros((1, H * g), dtype=torch.float32).pin_memory()
            o, l = ot.numpy(), lt.numpy()
            pin = [torch.from_numpy(x.view(np.int16)).pin_memory() for x in (qb, kb, vb)]
            qb, kb, vb = (t.numpy().view(np.uint16) for t in pin)
        c.decode_step_host(qb, kb, vb, o, lse=l)
        outs.append(o.copy())
        lses.append(l.copy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    assert np.array_equal(lses[0], lses[1]) and np.array_equal(lses[0], lses[2])


def test_sequence_sharded_attend_and_lse_merge():
    """Two R-aligned shards attended separately + LSE merge == one cache."""
    import torch

    from paper_2605_19660_b200 import KvCache, PipelineConfig, lse_merge

    H, g, S = 2, 4, 640
    k, v = make_inputs(11, S, H)
    q = dev_bf16(make_queries(11, 1, H * g))
    full = KvCache(PipelineConfig(heads=H), batch=1, q_heads=H * g, max_tokens=S + 8)
    full.buffer_quant(dev_bf16(k[None]), dev_bf16(v[None]))
    o_full, l_full = full.attend(q)
    parts_o, parts_l = [], []
    for lo, hi in ((0, 384), (384, S)):
        c = KvCache(PipelineConfig(heads=H), batch=1, q_heads=H * g, max_tokens=S)
        c.buffer_quant(dev_bf16(k[None, lo:hi]), dev_bf16(v[None, lo:hi]))
        o, l = c.attend(q)
        parts_o.append(o.reshape(H * g, 128))
        parts_l.append(l.reshape(H * g))
    merged = lse_merge(torch.stack(parts_o), torch.stack(parts_l))
    torch.cuda.synchronize()
    assert rel_err(merged.cpu().numpy(), o_full.reshape(H * g, 128).cpu().numpy()) < 1e-5


def test_decode_step_many_equals_per_cache_calls():
    """oscar_kv_decode_step_many (one host call for several caches, e.g. the
    layers of a step) == the same decode_step calls one by one, bit for bit."""
    import torch

    from paper_2605_19660_b200 import DecodeBatch, KvCache, PipelineConfig

    H, g, S, L = 2, 4, 260, 3
    data = [make_inputs(300 + i, S + 2, H) for i in range(L)]
    q = dev_bf16(make_queries(300, 1, H * g))

    def build():
        cs = []
        for k, v in data:
            c = KvCache(PipelineConfig(heads=H), batch=1, q_heads=H * g, max_tokens=S + 8)
            c.buffer_quant(dev_bf16(k[None, :S]), dev_bf16(v[None, :S]))
            cs.append(c)
        return cs

    one = build()
    ref = [c.decode_step(q, dev_bf16(d[0][S][None]), dev_bf16(d[1][S][None])) for c, d in zip(one, data)]
    many = build()
    outs = [torch.empty_like(r) for r in ref]
    DecodeBatch(many, [q] * L, [dev_bf16(d[0][S][None]) for d in data], [dev_bf16(d[1][S][None]) for d in data],
                outs).run()
    torch.cuda.synchronize()
    for a, b in zip(ref, outs):
        assert torch.equal(a, b)
    assert all(c.total_tokens == S + 1 for c in many)


def test_quantizer_exact_half_ties_bitexact():
    """Values landing exactly on half-integers of x/delta (llround's
    half-away-from-zero ties, quant.cpp:53-57) take the exact-division path of
    the device quantizer: codes must still equal the reference's."""
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H, S = 1, 256
    rng = np.random.default_rng(5)
    k, _ = make_inputs(21, S, H)
    # value groups of {0, 3, +-0.5, 1.5, 2.5, ...}: delta = 1, x/delta hits .5 ties
    choices = np.array([0.0, 3.0, 0.5, 1.5, 2.5, 1.0, 2.0, -0.0])
    v = rng.choice(choices, size=(S, H, 128))
    v[:, :, 0] = 0.0
    v[:, :, 1] = 3.0
    for bits in (2, 4):
        c = KvCache(PipelineConfig(heads=H, bits=bits, method="kivi"), batch=1, q_heads=H, max_tokens=S + 8)
        c.buffer_quant(dev_bf16(k[None]), dev_bf16(v[None]))
        o = ob.PortCache(method="kivi", bits=bits, H=H)
        o.append(k, v)
        assert ob.caches_equal(export_to_oracle(c.export(0), H), o.export()) == []


@pytest.mark.parametrize("bits,rotv", [(2, False), (4, False), (0, False), (2, True)])
def test_chunked_appends_equal_token_by_token(bits, rotv):
    """Streaming quantize-on-append: appending chunks of any size after the
    prefill (the decode branch of buffer_quant_k/v, kv_cache.cpp:219-249) gives
    the cache that token-by-token appends give -- whole R-blocks inside a chunk
    are quantized straight from the input -- and the oracle's cache."""
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H = 2
    chunks = [1, 50, 300, 7, 500, 128, 129, 3]
    S0, S = 200, 200 + sum(chunks)
    k, v = make_inputs(88 + bits, S, H)
    cfg = PipelineConfig(heads=H, bits=bits, rotate_v=rotv)
    a = KvCache(cfg, batch=1, q_heads=H, max_tokens=S + 8)
    a.buffer_quant(dev_bf16(k[None, :S0]), dev_bf16(v[None, :S0]))
    o = ob.PortCache(H=H, bits=bits, rotate_v=rotv)
    o.append(k[:S0], v[:S0])
    pos = S0
    for n in chunks:
        a.buffer_quant(dev_bf16(k[None, pos:pos + n]), dev_bf16(v[None, pos:pos + n]))
        o.append(k[pos:pos + n], v[pos:pos + n])
        pos += n
    assert (a.packed_tokens, a.residual_tokens) == ((S // 128) * 128, S % 128)
    assert ob.caches_equal(export_to_oracle(a.export(0), H), o.export()) == []
