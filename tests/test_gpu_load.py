"""KVC1 import on the device (KvCache::load, kv_cache.cpp:509-549; SURVEY.md
§8(f) #1): a cache dumped by the reference itself or by the device, loaded
into a fresh device cache, must export / re-dump byte-identically and attend
exactly like the cache that wrote it."""
import os
import tempfile

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2605_19660_b200.synthetic import make_inputs, make_queries

from gpu_util import dev_bf16, export_to_oracle, rel_err

pytestmark = pytest.mark.gpu

CASES = [  # method, bits, scaling, rotate_v, H
    ("oscar", 2, "l2", False, 2),
    ("oscar", 4, "rsqrt", False, 1),
    ("kivi", 2, "l2", False, 1),
    ("oscar", 0, "l2", False, 2),
    ("oscar", 2, "l2", True, 1),
    ("scale-only", 2, "mean-abs", False, 1),
]


def _ids(c):
    return "-".join(map(str, c))


@pytest.mark.parametrize("case", CASES, ids=_ids)
def test_device_dump_load_roundtrip(case):
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    method, bits, scaling, rotv, H = case
    cfg = PipelineConfig(method=method, bits=bits, scaling=scaling, heads=H, rotate_v=rotv)
    g, S = 4, 300
    k, v = make_inputs(61, S + 2, H)
    q = dev_bf16(make_queries(61, 1, H * g))
    a = KvCache(cfg, batch=1, q_heads=H * g, max_tokens=512)
    a.buffer_quant(dev_bf16(k[None, :S]), dev_bf16(v[None, :S]))
    with tempfile.TemporaryDirectory() as td:
        pa, pb = os.path.join(td, "a.kvc1"), os.path.join(td, "b.kvc1")
        a.dump(0, pa)
        b = KvCache(cfg, batch=1, q_heads=H * g, max_tokens=512)
        b.load(0, pa)
        assert (b.packed_tokens, b.residual_tokens, b.flush_count) == (a.packed_tokens, a.residual_tokens,
                                                                        a.flush_count)
        b.dump(0, pb)
        assert open(pa, "rb").read() == open(pb, "rb").read()
    # the loaded records are the written records: identical attention, bit for bit
    oa = a.decode_step(q, dev_bf16(k[None, S]), dev_bf16(v[None, S])).cpu().numpy()
    ob_ = b.decode_step(q, dev_bf16(k[None, S]), dev_bf16(v[None, S])).cpu().numpy()
    assert np.array_equal(oa, ob_)


@pytest.mark.parametrize("bits", [2, 4, 0])
def test_reference_dump_loads_on_device(bits):
    """A cache built and dumped by the reference's own C++ (KvCache::dump) is
    loaded on the device: export == the reference's export bit for bit, and a
    decode step matches the oracle's decode step over that cache."""
    if not ob.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H, g, S = 2, 4, 390
    k, v = make_inputs(70 + bits, S + 1, H)
    ref = ob.RefCache(H=H, bits=bits)
    ref.append(k[:S - 10], v[:S - 10])
    for t in range(S - 10, S):
        ref.append(k[t:t + 1], v[t:t + 1])
    c = KvCache(PipelineConfig(heads=H, bits=bits), batch=1, q_heads=H * g, max_tokens=S + 8)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "ref.kvc1")
        ref.dump(p)
        c.load(0, p)
        theirs = ref.export(td)
    assert ob.caches_equal(export_to_oracle(c.export(0), H), theirs) == []
    q = make_queries(70 + bits, 1, H * g)[0]
    port = ob.PortCache(H=H, bits=bits)
    port.append(k[:S - 10], v[:S - 10])
    for t in range(S - 10, S):
        port.append(k[t:t + 1], v[t:t + 1])
    want = port.decode_step(q, k[S], v[S], g)
    got = c.decode_step(dev_bf16(q[None]), dev_bf16(k[None, S]), dev_bf16(v[None, S])).cpu().numpy()[0]
    assert rel_err(got.astype(np.float64), want) <= (5e-3 if bits else 1e-2)


def test_load_rejects_mismatched_config():
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    H = 1
    k, v = make_inputs(80, 200, H)
    a = KvCache(PipelineConfig(heads=H, bits=2), batch=1, q_heads=H, max_tokens=256)
    a.buffer_quant(dev_bf16(k[None]), dev_bf16(v[None]))
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "a.kvc1")
        a.dump(0, p)
        b = KvCache(PipelineConfig(heads=H, bits=4), batch=1, q_heads=H, max_tokens=256)
        with pytest.raises(ValueError):
            b.load(0, p)
        small = KvCache(PipelineConfig(heads=H, bits=2), batch=1, q_heads=H, max_tokens=100)
        with pytest.raises(ValueError):
            small.load(0, p)
