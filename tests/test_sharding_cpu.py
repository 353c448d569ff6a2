"""Multi-GPU launcher logic on CPU: shard plans, the
bit-exactness of R-aligned sequence shards against the single cache (oracle),
and the (O, LSE) all-gather + log-sum-exp merge over a world_size-2 gloo
group.  The device merge kernel itself is covered by the GPU tests."""
import os

import numpy as np
import pytest

from oracle import bindings as ob
from paper_2605_19660_b200 import sharding as sh
from paper_2605_19660_b200.synthetic import make_inputs, make_queries

R = 128


@pytest.mark.parametrize("S,world", [(0, 2), (100, 2), (640, 2), (700, 3), (524288 + 77, 8), (4096, 8), (300, 8)])
def test_sequence_plan_is_r_aligned_partition(S, world):
    shards = [sh.sequence_shard(S, world, r) for r in range(world)]
    assert shards[0].tok_lo == 0 and shards[-1].tok_hi == S
    for a, b in zip(shards, shards[1:]):
        assert a.tok_hi == b.tok_lo
    for s in shards[:-1]:
        assert s.tok_lo % R == 0 and s.tok_hi % R == 0 and not s.tail
    assert shards[-1].tail and shards[-1].tok_lo % R == 0
    # the residual window lives on the tail, exactly as in the single cache
    assert shards[-1].tokens % R == S % R
    # packed blocks are balanced to within one block
    nb = [s.tokens // R for s in shards]
    assert max(nb) - min(nb) <= 1


def test_batch_and_head_plans():
    for B, world in [(16, 8), (256, 8), (3, 2), (1, 1)]:
        rs = [sh.batch_shard(B, world, r) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == B and all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    for Hkv, Hq, world in [(8, 32, 8), (4, 28, 4), (8, 32, 2), (4, 28, 2)]:
        hs = [sh.head_shard(Hkv, Hq, world, r) for r in range(world)]
        g = Hq // Hkv
        assert hs[0].kv_lo == 0 and hs[-1].kv_hi == Hkv and hs[-1].q_hi == Hq
        for x in hs:
            assert x.q_lo == x.kv_lo * g and x.q_hi == x.kv_hi * g
    with pytest.raises(ValueError):
        sh.head_shard(4, 28, 8, 0)
    with pytest.raises(ValueError):
        sh.head_shard(4, 30, 2, 0)


@pytest.mark.parametrize("S,world", [(700, 3), (1100, 2)])
def test_sequence_shards_union_equals_single_cache(S, world):
    """Per-rank caches built from R-aligned slices are the single cache's
    blocks, bit for bit (codes, steps, zero points, norms, residual)."""
    H = 2
    k, v = make_inputs(31, S + 5, H)
    full = ob.PortCache(H=H)
    full.append(k[:S], v[:S])
    parts = []
    for r in range(world):
        s = sh.sequence_shard(S, world, r)
        c = ob.PortCache(H=H)
        c.append(k[s.tok_lo:s.tok_hi], v[s.tok_lo:s.tok_hi])
        if s.tail:  # streaming appends land on the tail and flush where the single cache flushes
            for t in range(S, S + 5):
                c.append(k[t:t + 1], v[t:t + 1])
        parts.append(c)
    for t in range(S, S + 5):
        full.append(k[t:t + 1], v[t:t + 1])
    kf, vf = full.materialize()
    ks, vs = zip(*(c.materialize() for c in parts))
    assert np.array_equal(np.concatenate(ks), kf) and np.array_equal(np.concatenate(vs), vf)
    assert sum(c.stats()["packed"] for c in parts) == full.stats()["packed"]
    assert parts[-1].stats()["residual"] == full.stats()["residual"]


def _partial(q_rot, kmat, vmat, g):
    """(O, LSE) of GQA attention over one shard (fp64), test helper."""
    Hq, d = q_rot.shape
    o = np.zeros((Hq, d))
    lse = np.full(Hq, -np.inf)
    if kmat.shape[0] == 0:
        return o, lse
    for j in range(Hq):
        lg = kmat[:, j // g, :] @ q_rot[j] / np.sqrt(d)
        m = lg.max()
        w = np.exp(lg - m)
        o[j] = (w / w.sum()) @ vmat[:, j // g, :]
        lse[j] = m + np.log(w.sum())
    return o, lse


def _merge(outs, lses):
    M = lses.max(axis=0)
    w = np.where(np.isinf(lses), 0.0, np.exp(lses - M))
    return (w[:, :, None] * outs).sum(0) / w.sum(0)[:, None]


def _worker(rank, world, rdzv, S, H, g, q, res_path):
    import torch
    import torch.distributed as td

    td.init_process_group("gloo", init_method=f"file://{rdzv}", rank=rank, world_size=world)
    try:
        k, v = make_inputs(41, S, H)
        s = sh.sequence_shard(S, world, rank)
        c = ob.PortCache(H=H)
        c.append(k[s.tok_lo:s.tok_hi], v[s.tok_lo:s.tok_hi])
        km, vm = c.materialize()
        qr = np.stack([ob.port_fht(x) for x in q])
        o, l = _partial(qr, km, vm, g)
        outs, lses = sh.gather_partials(torch.from_numpy(o).float(), torch.from_numpy(l).float())
        assert outs.shape == (world, H * g, 128) and lses.shape == (world, H * g)
        merged = _merge(outs.double().numpy(), lses.double().numpy())
        if rank == 0:
            np.save(res_path, merged)
    finally:
        td.destroy_process_group()


def test_gloo_world2_gather_and_lse_merge(tmp_path):
    """Two ranks attend their R-aligned shards, all-gather (O, LSE) over gloo,
    and the log-sum-exp merge equals attention over the whole cache."""
    import torch.multiprocessing as mp

    S, H, g, world = 900, 2, 4, 2
    q = make_queries(41, 1, H * g)[0]
    res = str(tmp_path / "merged.npy")
    mp.spawn(_worker, args=(world, str(tmp_path / "rdzv"), S, H, g, q, res), nprocs=world, join=True)
    merged = np.load(res)
    k, v = make_inputs(41, S, H)
    full = ob.PortCache(H=H)
    full.append(k, v)
    km, vm = full.materialize()
    ref = ob.port_attention(np.stack([ob.port_fht(x) for x in q])[None],
                            np.repeat(km, g, axis=1), np.repeat(vm, g, axis=1))[0]
    # fp32 exchange of fp64 partials: agreement to fp32 rounding
    assert np.max(np.abs(merged - ref)) / np.max(np.abs(ref)) < 1e-6
