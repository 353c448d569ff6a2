"""Pin the CPU oracle (oracle/oscar_oracle.c) against the reference.

Three anchors:
  * the reference's own known answers (test_quant.cpp, test_kv_cache.cpp,
    test_hadamard.cpp, test_pipeline.cpp) re-expressed here;
  * the compiled reference itself (oracle/_ref), bit-exact, when present;
  * committed golden fixtures in tests/golden/ (generated from oracle/_ref by
    tests/golden/make_golden.py), so the pin also holds where
    /root/reference is absent.
"""
import glob
import math
import os
import tempfile

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2605_19660_b200.synthetic import make_inputs, make_queries, round_bf16

needs_ref = pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---- known answers ---------------------------------------------------------
def test_pack_word_golden_e4e4():
    # test_quant.cpp:206-218
    w = ob.port_pack_2bit([0, 1, 2, 3, 0, 1, 2, 3])
    assert w.tolist() == [0xE4E4]
    assert ob.port_pack_2bit([0] * 16).tolist() == [0, 0]


def test_quant_params_hand_cases():
    # test_quant.cpp:13-26
    assert ob.port_quant_params([0, 1, 2, 3], 2) == (1.0, 0, 0.0)
    d, zp, _ = ob.port_quant_params([-1, 1], 2)
    assert abs(d - 2.0 / 3.0) < 1e-15 and zp == 2  # round(1.5) away from zero
    d, zp, c = ob.port_quant_params([5, 5, 5], 2)
    assert (d, zp, c) == (0.0, 0, 5.0)
    L = ob.Port.lib()
    assert L.oo_dequantize_one(0, 0.0, 0, 5.0) == 5.0


def test_zero_point_not_clamped():
    # test_quant.cpp:51-65 (code wins over SPEC)
    d, zp, _ = ob.port_quant_params([5, 6, 7, 8], 2)
    assert zp < 0
    L = ob.Port.lib()
    for x in (5, 6, 7, 8):
        q = L.oo_quantize_one(x, d, zp, 2)
        assert abs(L.oo_dequantize_one(q, d, zp, 5.0) - x) < 1e-12
    d, zp, _ = ob.port_quant_params([-8, -7, -6, -5], 2)
    assert zp > 3


def test_fht_hand_vectors():
    # test_hadamard.cpp:13-27
    v = ob.port_fht([1.0, 1.0])
    assert abs(v[0] - math.sqrt(2)) < 1e-15 and abs(v[1]) < 1e-15
    assert np.allclose(ob.port_fht([1.0, 0, 0, 0]), 0.5, atol=1e-15)


def test_scale_hand_values():
    # test_pipeline.cpp:102-116, 132-139
    sc, nr, deg = ob.port_token_scale(np.array([[[3.0, 4.0]]]), "l2")
    assert abs(nr[0] - 5.0) < 1e-15 and abs(sc[0, 0, 0] - 0.6) < 1e-15
    sc, nr, _ = ob.port_token_scale(np.ones((1, 1, 4)), "max")
    assert nr[0] == 1.0
    x = np.zeros((2, 1, 4))
    x[1, 0, 0] = 1.0
    _, nr, deg = ob.port_token_scale(x, "l2")
    assert deg == 1 and nr[0] == 1e-12 and nr[1] == 1.0


def test_prefill_split_and_flush_counts():
    # test_kv_cache.cpp:59-93
    k, v = make_inputs(31, 300, 2, 64)
    c = ob.PortCache(H=2, d=64)
    c.append(k, v)
    assert c.stats() == dict(packed=256, residual=44, total=300, flushes=0)
    c = ob.PortCache(H=2, d=64)
    k, v = make_inputs(35, 127, 2, 64)
    c.append(k, v)
    k1, v1 = make_inputs(37, 1, 2, 64)
    c.append(k1, v1)
    assert c.stats() == dict(packed=128, residual=0, total=128, flushes=1)


def test_invalid_configs_rejected():
    # test_kv_cache.cpp:47-57
    with pytest.raises(ValueError):
        ob.PortCache(H=2, d=64, R=100)
    with pytest.raises(ValueError):
        ob.PortCache(H=2, d=64, bits=5)
    with pytest.raises(ValueError):
        ob.PortCache(H=2, d=48)


def test_flush_consistency_batched_equals_stepped():
    # test_kv_cache.cpp:137-176, acceptance crit 4
    for S, R in ((300, 128), (256, 128), (130, 64)):
        k, v = make_inputs(41, S, 2, 64)
        a = ob.PortCache(H=2, d=64, R=R)
        a.append(k, v)
        b = ob.PortCache(H=2, d=64, R=R)
        b.append(k[:0], v[:0])
        for t in range(S):
            b.append(k[t : t + 1], v[t : t + 1])
        ka, va = a.materialize()
        kb, vb = b.materialize()
        assert np.max(np.abs(ka - kb)) <= 1e-12 and np.max(np.abs(va - vb)) <= 1e-12


# ---- bit-exact against the compiled reference --------------------------------
CONFIGS = [
    # method, bits, scaling, S, H, d, R, rotate_v
    ("oscar", 2, "l2", 300, 2, 128, 128, False),
    ("oscar", 2, "rsqrt", 300, 2, 128, 128, False),
    ("oscar", 4, "l2", 300, 2, 128, 128, False),
    ("oscar", 2, "max", 200, 2, 64, 64, False),
    ("oscar", 2, "mean-abs", 200, 1, 64, 128, True),
    ("kivi", 2, "l2", 260, 2, 128, 128, False),
    ("rotate-only", 2, "l2", 130, 2, 64, 64, False),
    ("scale-only", 4, "l2", 130, 2, 64, 64, False),
    ("oscar", 0, "l2", 140, 2, 64, 128, False),
    ("oscar", 8, "l2", 140, 2, 64, 128, False),
]


@needs_ref
@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: "-".join(map(str, c)))
def test_port_matches_reference_bitexact(cfg):
    method, bits, scaling, S, H, d, R, rotv = cfg
    k, v = make_inputs(hash(cfg) % 1000, S, H, d)
    kw = dict(method=method, bits=bits, scaling=scaling, d=d, H=H, R=R, rotate_v=rotv)
    ref = ob.RefCache(**kw)
    port = ob.PortCache(**kw)
    # prefill S-7, then 7 single-token appends (crosses no or one flush)
    ref.append(k[: S - 7], v[: S - 7])
    port.append(k[: S - 7], v[: S - 7])
    for t in range(S - 7, S):
        ref.append(k[t : t + 1], v[t : t + 1])
        port.append(k[t : t + 1], v[t : t + 1])
    with tempfile.TemporaryDirectory() as td:
        er = ref.export(td)
    ep = port.export()
    assert ob.caches_equal(er, ep) == []
    kr, vr = ref.materialize()
    kp, vp = port.materialize()
    assert np.array_equal(kr, kp) and np.array_equal(vr, vp)


@needs_ref
def test_port_decode_step_matches_reference():
    H, g, d = 2, 4, 128
    k, v = make_inputs(5, 257, H, d)
    q = make_queries(5, 3, H * g, d)
    ref = ob.RefCache(H=H, d=d)
    port = ob.PortCache(H=H, d=d)
    ref.append(k[:255], v[:255])
    port.append(k[:255], v[:255])
    for i, t in enumerate((255, 256)):
        o_r = ref.decode_step(q[i], k[t], v[t], g)
        o_p = port.decode_step(q[i], k[t], v[t], g)
        assert np.array_equal(o_r, o_p)


@needs_ref
def test_port_attention_and_scale_match_reference():
    rng = np.random.default_rng(3)
    q, kk, vv = rng.standard_normal((3, 2, 16)), rng.standard_normal((24, 2, 16)), rng.standard_normal((24, 2, 16))
    assert np.array_equal(ob.ref_attention(q, kk, vv), ob.port_attention(q, kk, vv))
    x = round_bf16(rng.standard_normal((64, 3, 128)) * 3)
    for s in ("l2", "rsqrt", "max", "mean-abs"):
        a, b = ob.ref_token_scale(x, s), ob.port_token_scale(x, s)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert ob.ref_pack_2bit([0, 1, 2, 3, 0, 1, 2, 3]).tolist() == [0xE4E4]


# ---- golden fixtures (travel with the repo; no /root/reference needed) -------
def _golden_files():
    return sorted(glob.glob(os.path.join(GOLDEN, "cache_*.npz")))


def export_to_flat(ec: ob.ExportedCache) -> dict:
    """Flatten an exported cache to the arrays stored in golden fixtures."""
    out = {}
    for kind, blocks in (("k", ec.k_blocks), ("v", ec.v_blocks)):
        for f in ("codes", "delta", "zp", "constant", "raw"):
            arrs = [np.asarray(b[f]) for h in blocks for b in h]
            out[f"{kind}_{f}"] = np.concatenate(arrs) if arrs else np.zeros(0)
    out["k_norms"] = np.concatenate(ec.k_norms) if ec.k_norms else np.zeros(0)
    out["k_residual"] = ec.k_residual.reshape(-1)
    out["k_norms_residual"] = ec.k_norms_residual
    out["v_residual"] = ec.v_residual.reshape(-1)
    out["stats"] = np.array([ec.packed_tokens, ec.residual_tokens, ec.flush_count], np.int64)
    return out


@pytest.mark.parametrize("path", _golden_files(), ids=os.path.basename)
def test_port_matches_golden(path):
    g = np.load(path, allow_pickle=False)
    meta = {k[5:]: g[k].item() for k in g.files if k.startswith("meta_")}
    port = ob.PortCache(method=str(g["method"]), bits=int(meta["bits"]), scaling=str(g["scaling"]),
                        d=int(meta["d"]), H=int(meta["H"]), R=int(meta["R"]), rotate_v=bool(meta["rotate_v"]))
    k, v = g["k_in"], g["v_in"]
    cut = int(meta["prefill"])
    port.append(k[:cut], v[:cut])
    for t in range(cut, k.shape[0]):
        port.append(k[t : t + 1], v[t : t + 1])
    flat = export_to_flat(port.export())
    for name, arr in flat.items():
        exp = g["x_" + name]
        assert arr.shape == exp.shape and np.array_equal(
            np.ascontiguousarray(arr).view(np.uint8), np.ascontiguousarray(exp.astype(arr.dtype)).view(np.uint8)
        ), name
    if "q_in" in g.files:
        q = g["q_in"]
        o = port.decode_step(q, g["k_cur"], g["v_cur"], int(meta["gqa"]), append=False)
        assert np.array_equal(o, g["x_decode_out"])
