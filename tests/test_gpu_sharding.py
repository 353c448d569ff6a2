"""Multi-rank paths through the CUDA library.

The GPU box has one B200, so the SPMD code runs as two gloo ranks sharing
cuda:0 (NCCL refuses two ranks on one device); the exchange is the same
gather_partials call the NCCL launcher makes, the merge is the device
log-sum-exp kernel.  Reference semantics: the sharded result must equal one
cache holding the whole context (up to fp16 softmax-weight rounding, SHARD_TOL)."""
import os

import numpy as np
import pytest

from gpu_util import dev_bf16, rel_err

pytestmark = pytest.mark.gpu

S, H, G_, STEPS = 1000, 2, 4, 30  # residual 104 -> the 24th decode step flushes on the tail rank
# shards vs one cache: the residual-window tile seeds the running max of the warp that
# takes it, and which packed units share a warp with it follows the stream-K split of
# the launch, so the fp16 softmax weights P are rounded against different maxima on
# the two sides (fp16 P rounding, ~1e-4); both are within the stated 5e-3 of the oracle
SHARD_TOL = 5e-4


def _inputs():
    from paper_2605_19660_b200.synthetic import make_inputs, make_queries

    k, v = make_inputs(77, S + STEPS, H)
    q = make_queries(77, STEPS, H * G_)
    return k, v, q


def _seq_worker(rank, world, rdzv, res_path, side_stream=False):
    import torch
    import torch.distributed as td

    from paper_2605_19660_b200 import PipelineConfig
    from paper_2605_19660_b200.sharding import SeqShardedKvCache

    torch.cuda.set_device(0)
    td.init_process_group("gloo", init_method=f"file://{rdzv}", rank=rank, world_size=world)
    try:
        k, v, q = _inputs()
        c = SeqShardedKvCache(PipelineConfig(heads=H), batch=1, q_heads=H * G_, max_tokens_per_rank=S + STEPS)
        c.prefill(dev_bf16(k[None, :S]), dev_bf16(v[None, :S]))
        outs = []
        st = torch.cuda.Stream() if side_stream else None
        for t in range(STEPS):
            qt, kt, vt = dev_bf16(q[t][None]), dev_bf16(k[S + t][None]), dev_bf16(v[S + t][None])
            if st is None:
                o = c.decode_step(qt, kt, vt)
            else:
                # a NON-current stream, held back by a spin kernel: the exchange and
                # merge must be ordered after the attention kernel on that stream
                st.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(st):
                    torch.cuda._sleep(2_000_000)
                o = c.decode_step(qt, kt, vt, stream=st.cuda_stream)
                torch.cuda.current_stream().wait_stream(st)
            outs.append(o.cpu().numpy())
        tot = c.total_tokens
        if rank == 0:
            np.save(res_path, np.stack(outs))
        assert tot == S + STEPS
        c.close()
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("side_stream", [False, True])
def test_sequence_sharded_decode_matches_single_cache(tmp_path, side_stream):
    import torch.multiprocessing as mp

    from paper_2605_19660_b200 import KvCache, PipelineConfig

    res = str(tmp_path / "seq.npy")
    mp.spawn(_seq_worker, args=(2, str(tmp_path / "rdzv"), res, side_stream), nprocs=2, join=True)
    sharded = np.load(res)
    k, v, q = _inputs()
    c = KvCache(PipelineConfig(heads=H), batch=1, q_heads=H * G_, max_tokens=S + STEPS)
    c.buffer_quant(dev_bf16(k[None, :S]), dev_bf16(v[None, :S]))
    for t in range(STEPS):
        o = c.decode_step(dev_bf16(q[t][None]), dev_bf16(k[S + t][None]), dev_bf16(v[S + t][None])).cpu().numpy()
        assert rel_err(sharded[t], o) < SHARD_TOL, t
    assert c.flush_count == 1


def test_head_sharded_equals_full_heads():
    """KV heads [h0, h1) + their query heads on their own cache == the same
    heads of the full cache (C4 partitioning, no communication)."""
    import torch

    from paper_2605_19660_b200 import KvCache, PipelineConfig
    from paper_2605_19660_b200.sharding import head_shard
    from paper_2605_19660_b200.synthetic import make_inputs, make_queries

    B, Hkv, g, Sx = 2, 4, 7, 700
    data = [make_inputs(90 + b, Sx + 1, Hkv) for b in range(B)]
    k = np.stack([d[0] for d in data])
    v = np.stack([d[1] for d in data])
    q = np.stack([make_queries(90 + b, 1, Hkv * g)[0] for b in range(B)])
    full = KvCache(PipelineConfig(heads=Hkv), batch=B, q_heads=Hkv * g, max_tokens=Sx + 4)
    full.buffer_quant(dev_bf16(k[:, :Sx]), dev_bf16(v[:, :Sx]))
    of = full.decode_step(dev_bf16(q), dev_bf16(k[:, Sx]), dev_bf16(v[:, Sx])).cpu().numpy()
    for rank in range(2):
        hs = head_shard(Hkv, Hkv * g, 2, rank)
        c = KvCache(PipelineConfig(heads=hs.kv_hi - hs.kv_lo), batch=B, q_heads=hs.q_hi - hs.q_lo,
                    max_tokens=Sx + 4)
        c.buffer_quant(dev_bf16(k[:, :Sx, hs.kv_lo:hs.kv_hi]), dev_bf16(v[:, :Sx, hs.kv_lo:hs.kv_hi]))
        o = c.decode_step(dev_bf16(q[:, hs.q_lo:hs.q_hi]), dev_bf16(k[:, Sx, hs.kv_lo:hs.kv_hi]),
                          dev_bf16(v[:, Sx, hs.kv_lo:hs.kv_hi])).cpu().numpy()
        torch.cuda.synchronize()
        assert rel_err(o, of[:, hs.q_lo:hs.q_hi]) < SHARD_TOL
        # the packed blocks are the full cache's blocks, bit for bit
        ef, eh = full.export(1), c.export(1)
        for key in ("k_payload", "v_payload", "k_delta", "k_zp", "v_delta", "v_zp", "k_norms"):
            assert np.array_equal(eh[key], ef[key][hs.kv_lo:hs.kv_hi]), key


# ---------------------------------------------------------------- fused peer-memory exchange
def _single_cache_outputs(cfg=None):
    from paper_2605_19660_b200 import KvCache, PipelineConfig

    k, v, q = _inputs()
    c = KvCache(cfg or PipelineConfig(heads=H), batch=1, q_heads=H * G_, max_tokens=S + STEPS)
    c.buffer_quant(dev_bf16(k[None, :S]), dev_bf16(v[None, :S]))
    return [c.decode_step(dev_bf16(q[t][None]), dev_bf16(k[S + t][None]), dev_bf16(v[S + t][None])).cpu().numpy()
            for t in range(STEPS)]


@pytest.mark.parametrize("world,bits,rotate_v", [(2, 2, False), (3, 2, False), (2, 4, True)])
def test_peer_publish_merge_virtual_ranks(world, bits, rotate_v):
    """The attention kernel publishes its rows into every rank's receive area
    and the flag-polling merge kernel combines them (oscar_kv_attend_publish +
    oscar_peer_merge).  `world` virtual ranks share cuda:0 (their areas are
    mapped directly); publish kernels go first on the stream, then the merges.
    30 steps (epoch parities alternate) crossing a flush on the tail shard."""
    import torch

    from paper_2605_19660_b200 import KvCache, PipelineConfig
    from paper_2605_19660_b200 import kv_cache as kc
    from paper_2605_19660_b200.sharding import local_peer_plans, sequence_shard

    k, v, q = _inputs()
    rows = H * G_
    cfg = PipelineConfig(heads=H, bits=bits, rotate_v=rotate_v)
    plans, areas = local_peer_plans(world, rows)
    shards = [sequence_shard(S, world, r) for r in range(world)]
    caches = []
    for sh in shards:
        c = KvCache(cfg, batch=1, q_heads=rows, max_tokens=S + STEPS)
        c.buffer_quant(dev_bf16(k[None, sh.tok_lo:sh.tok_hi]), dev_bf16(v[None, sh.tok_lo:sh.tok_hi]))
        caches.append(c)
    ref = _single_cache_outputs(cfg)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    outs = [torch.empty((rows, 128), dtype=torch.float32, device="cuda") for _ in range(world)]
    lses = [torch.empty((rows,), dtype=torch.float32, device="cuda") for _ in range(world)]
    for t in range(STEPS):
        epoch = t + 1
        qt, kt, vt = dev_bf16(q[t][None]), dev_bf16(k[S + t][None]), dev_bf16(v[S + t][None])
        for r, (c, sh) in enumerate(zip(caches, shards)):
            if sh.tail:
                c.attend_publish(qt, plans[r], epoch, kt, vt)
            else:
                c.attend_publish(qt, plans[r], epoch)
        for r in range(world):
            kc.peer_merge(plans[r], epoch, outs[r], lses[r], status)
        for r in range(world):
            assert rel_err(outs[r].cpu().numpy()[None], ref[t]) < SHARD_TOL, (t, r)
    assert status.item() == 0
    assert caches[-1].flush_count == 1
    # every rank merged the same rows; LSE equals the single cache's
    full = KvCache(cfg, batch=1, q_heads=rows, max_tokens=S + STEPS + 1)
    full.buffer_quant(dev_bf16(k[None, :S + STEPS]), dev_bf16(v[None, :S + STEPS]))
    _, lse_full = full.attend(dev_bf16(q[STEPS - 1][None]))
    for r, c in enumerate(caches):
        c.attend_publish(dev_bf16(q[STEPS - 1][None]), plans[r], STEPS + 1)
    kc.peer_merge(plans[0], STEPS + 1, outs[0], lses[0], status)
    assert np.allclose(lses[0].cpu().numpy(), lse_full.cpu().numpy().ravel(), atol=2e-4)


def test_peer_publish_empty_shard_and_timeout():
    """An empty shard publishes LSE = -inf rows (no softmax mass); a rank whose
    peer never publishes gets status 1 and NaN rows after ~5 s, not a hang."""
    import torch

    from paper_2605_19660_b200 import KvCache, PipelineConfig
    from paper_2605_19660_b200 import kv_cache as kc
    from paper_2605_19660_b200.sharding import local_peer_plans

    k, v, q = _inputs()
    rows = H * G_
    plans, areas = local_peer_plans(2, rows)
    c = KvCache(PipelineConfig(heads=H), batch=1, q_heads=rows, max_tokens=S + 4)
    c.buffer_quant(dev_bf16(k[None, :S]), dev_bf16(v[None, :S]))
    o_ref, _ = c.attend(dev_bf16(q[0][None]))
    kc.peer_publish_empty(plans[0], 1)
    c.attend_publish(dev_bf16(q[0][None]), plans[1], 1)
    out = torch.empty((rows, 128), dtype=torch.float32, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    kc.peer_merge(plans[0], 1, out, None, status)
    assert status.item() == 0
    assert rel_err(out.cpu().numpy(), o_ref.cpu().numpy()[0]) < 1e-6
    kc.peer_merge(plans[0], 2, out, None, status)  # epoch 2 was never published
    assert status.item() == 1
    assert np.isnan(out.cpu().numpy()).all()


def _p2p_worker(rank, world, rdzv, res_path):
    import torch
    import torch.distributed as td

    from paper_2605_19660_b200 import PipelineConfig
    from paper_2605_19660_b200.sharding import SeqShardedKvCache

    torch.cuda.set_device(0)
    td.init_process_group("gloo", init_method=f"file://{rdzv}", rank=rank, world_size=world)
    try:
        k, v, q = _inputs()
        c = SeqShardedKvCache(PipelineConfig(heads=H), batch=1, q_heads=H * G_, max_tokens_per_rank=S + STEPS,
                              exchange="p2p")
        c.prefill(dev_bf16(k[None, :S]), dev_bf16(v[None, :S]))
        outs = []
        for t in range(8):
            o = c.decode_step(dev_bf16(q[t][None]), dev_bf16(k[S + t][None]), dev_bf16(v[S + t][None]))
            outs.append(o.cpu().numpy())
        np.save(res_path + f".{rank}.npy", np.stack(outs))
        td.barrier()
        c.close()
    finally:
        td.destroy_process_group()


def test_p2p_exchange_two_processes_ipc(tmp_path):
    """The SPMD p2p path end to end: two processes (gloo only for the one-time
    IPC handle exchange) map each other's receive areas with CUDA IPC; every
    step's rows travel by the attention kernels' peer stores.  Both share
    cuda:0 here (one B200 per box); on 8 GPUs the same stores go over NVLink."""
    import torch.multiprocessing as mp

    res = str(tmp_path / "p2p")
    mp.spawn(_p2p_worker, args=(2, str(tmp_path / "rdzv"), res), nprocs=2, join=True)
    ref = _single_cache_outputs()
    for rank in range(2):
        got = np.load(res + f".{rank}.npy")
        for t in range(8):
            assert rel_err(got[t], ref[t]) < SHARD_TOL, (rank, t)


def _nccl_gather_worker(rdzv, out_path):
    import numpy as np
    import torch
    import torch.distributed as td

    from paper_2605_19660_b200.kv_cache import lse_merge
    from paper_2605_19660_b200.sharding import gather_partials

    torch.cuda.set_device(0)
    td.init_process_group("nccl", init_method=f"file://{rdzv}", rank=0, world_size=1,
                          device_id=torch.device("cuda", 0))
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    o = torch.randn((28, 128), generator=g, device="cuda")
    lse = torch.randn((28,), generator=g, device="cuda")
    outs, lses = gather_partials(o, lse)  # the NCCL branch: all_gather_into_tensor of [rows, d+1]
    merged = lse_merge(outs, lses)
    torch.cuda.synchronize()
    assert td.get_backend() == "nccl"
    np.save(out_path, np.stack([o.cpu().numpy(), outs[0].cpu().numpy(), merged.cpu().numpy()]))
    td.destroy_process_group()


def test_nccl_gather_partials_branch(tmp_path):
    """gather_partials' NCCL branch (one packed all_gather_into_tensor of (O, LSE)) on a
    one-rank NCCL group on the B200 (the box has one GPU; NCCL rejects two ranks on one
    device), followed by the device LSE merge: a single partial merges to itself."""
    import multiprocessing as mp

    import numpy as np

    ctx = mp.get_context("spawn")
    out = tmp_path / "nccl.npy"
    p = ctx.Process(target=_nccl_gather_worker, args=(str(tmp_path / "rdzv"), str(out)))
    p.start()
    p.join(240)
    assert p.exitcode == 0, p.exitcode
    o, gathered, merged = np.load(out)
    assert np.array_equal(o, gathered)
    assert np.allclose(merged, o, rtol=1e-6, atol=1e-6)
