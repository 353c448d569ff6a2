"""Multi-GPU launcher for the OScaR KV-cache path.

One process per GPU (torch.distributed over NCCL for the plumbing).  Three
partitionings, matching BASELINE.json configs 3-5:

* batch sharding (C3): sequences [b0, b1) live on rank r, all KV heads --
  no communication (the reference has no cross-sequence term);
* head sharding (C4): KV heads [h0, h1) and their GQA query heads live on
  rank r -- no communication (attend_one has no cross-head term,
  pipeline.cpp:152-180; cache state is per head, kv_cache.hpp:111-116);
* sequence sharding (C5): the context is cut into R-aligned token ranges so
  that quantisation groups and R-blocks never straddle ranks (flush_k_block /
  flush_v_block work on whole R-blocks, kv_cache.cpp:101-157); the residual
  window and every appended token live on the tail rank, which therefore
  flushes exactly when the single-cache reference would.  Each rank attends
  its shard; the (O, LSE) partials are either exchanged with ONE all-gather
  and merged by oscar_lse_merge (exchange="nccl"), or published by the
  attention kernel itself into every rank's receive area over NVLink peer
  memory and merged by one flag-polling kernel (exchange="p2p",
  PeerExchange; no collective on the data path).

The reference is single-process (no MPI/NCCL anywhere); these
plans are new, but the union of the per-rank caches is bit-identical to the
single cache the reference would build (tests/test_sharding_cpu.py checks that
with the oracle).
"""
from __future__ import annotations

import contextlib
from dataclasses import dataclass

R = 128
D = 128


# ----------------------------------------------------------------------------- plans
def even_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of an even contiguous split of n items (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    return (rank * n) // world, ((rank + 1) * n) // world


def batch_shard(B: int, world: int, rank: int) -> tuple[int, int]:
    """Sequences of rank `rank` (C3)."""
    return even_range(B, world, rank)


@dataclass(frozen=True)
class HeadShard:
    kv_lo: int
    kv_hi: int
    q_lo: int
    q_hi: int


def head_shard(Hkv: int, Hq: int, world: int, rank: int) -> HeadShard:
    """KV heads [kv_lo, kv_hi) and their GQA query heads (C4).  Query head j
    attends KV head j // (Hq/Hkv), so a KV-head range owns a contiguous,
    group-aligned query range."""
    if Hq % Hkv:
        raise ValueError("q_heads must be a multiple of kv heads")
    if world > Hkv:
        raise ValueError(f"head sharding needs world ({world}) <= kv heads ({Hkv})")
    g = Hq // Hkv
    lo, hi = even_range(Hkv, world, rank)
    return HeadShard(lo, hi, lo * g, hi * g)


@dataclass(frozen=True)
class SeqShard:
    tok_lo: int      # first context token of this rank
    tok_hi: int      # one past the last prefill token of this rank
    tail: bool       # owns the residual window and all appended tokens

    @property
    def tokens(self) -> int:
        return self.tok_hi - self.tok_lo


def sequence_shard(S: int, world: int, rank: int, R_: int = R) -> SeqShard:
    """R-aligned token range of rank `rank` for a prefill of S tokens (C5).

    The S - S mod R packed tokens are split in whole R-blocks (even split of
    blocks); the S mod R residual tokens go to the last rank, exactly where
    the single cache keeps them (kv_cache.cpp:204-218)."""
    nblk = S // R_
    b0, b1 = even_range(nblk, world, rank)
    tail = rank == world - 1
    return SeqShard(b0 * R_, S if tail else b1 * R_, tail)


# ----------------------------------------------------------------------------- exchange
def _dist():
    import torch.distributed as td

    return td


def gather_partials(o, lse, group=None):
    """All-gather this rank's (O [rows, d] fp32, LSE [rows] fp32) partial.

    Both are packed into one [rows, d+1] buffer so the exchange is ONE
    collective (latency-bound: C5 moves 14.4 KB per rank per layer).  Returns
    (outs [P, rows, d], lses [P, rows]) on o's device.  Works on NCCL (CUDA
    tensors) and gloo (CPU tensors, the multi-process CPU tests)."""
    import torch

    td = _dist()
    rows, d = o.shape
    if not td.is_initialized():  # single process: nothing to exchange
        return o.reshape(1, rows, d), lse.reshape(1, rows)
    P = td.get_world_size(group)
    buf = torch.cat([o.reshape(rows, d), lse.reshape(rows, 1)], dim=1).contiguous()
    if td.get_backend(group) == "nccl":
        allb = torch.empty((P, rows, d + 1), dtype=buf.dtype, device=buf.device)
        td.all_gather_into_tensor(allb, buf, group=group)
    else:  # gloo: host staging (multi-process tests, several ranks sharing one GPU)
        hb = buf.cpu()
        parts = [torch.empty_like(hb) for _ in range(P)]
        td.all_gather(parts, hb, group=group)
        allb = torch.stack(parts).to(buf.device)
    return allb[:, :, :d].contiguous(), allb[:, :, d].contiguous()


class PeerExchange:
    """Receive areas of the fused sequence-shard exchange (oscar_kv_attend_publish
    + oscar_peer_merge): this rank allocates its area on its GPU, the 64-byte
    CUDA IPC handles are all-gathered over the process group (host bytes, so
    gloo or NCCL), and every peer's area is mapped here.  No collective runs on
    the data path: the attention kernel stores its rows into the peers' areas
    over NVLink and the merge kernel polls the local flags."""

    def __init__(self, rows: int, device: int = 0, group=None):
        from . import kv_cache as kc

        td = _dist()
        self.world = td.get_world_size(group) if td.is_initialized() else 1
        self.rank = td.get_rank(group) if td.is_initialized() else 0
        self.rows, self.device = rows, device
        nbytes = kc.peer_area_bytes(self.world, rows)
        self._own, handle = kc.ipc_alloc(nbytes, device)
        handles = [None] * self.world
        if self.world > 1:
            td.all_gather_object(handles, handle, group=group)
        else:
            handles = [handle]
        self._opened = []
        areas = []
        for p, h in enumerate(handles):
            if p == self.rank:
                areas.append(self._own)
            else:
                a = kc.ipc_open(h, device)
                self._opened.append(a)
                areas.append(a)
        self.plan = kc.PeerPlan(self.world, self.rank, rows, areas)
        self.epoch = 0

    def close(self):
        from . import kv_cache as kc

        for a in self._opened:
            kc.ipc_close(a)
        self._opened = []
        if self._own:
            kc.ipc_free(self._own)
            self._own = 0


def local_peer_plans(world: int, rows: int, device=None):
    """Receive areas of `world` VIRTUAL ranks on one device (single-GPU tests of
    the publish / merge kernels: every plan maps every area directly).
    Returns (plans, areas); keep `areas` alive while the plans are used."""
    import torch

    from . import kv_cache as kc

    nbytes = kc.peer_area_bytes(world, rows)
    areas = [torch.zeros(nbytes, dtype=torch.uint8, device=device or "cuda") for _ in range(world)]
    ptrs = [a.data_ptr() for a in areas]
    return [kc.PeerPlan(world, r, rows, ptrs) for r in range(world)], areas


# ----------------------------------------------------------------------------- sharded caches
class SeqShardedKvCache:
    """One rank's share of a sequence-sharded cache (C5).

    Every rank calls the same methods in the same order (SPMD).  prefill()
    takes the FULL context tensors [B, S, H, d] or just this rank's slice
    (pass `sliced=True`); decode_step() returns the merged attention output of
    the whole context (+ current token) on every rank.
    """

    def __init__(self, cfg, batch: int, q_heads: int, max_tokens_per_rank: int, device: int = 0,
                 keep_exact: bool = True, group=None, merge=None, exchange: str = "nccl", strict: bool = True):
        """exchange: "nccl" (all-gather of the packed partials + lse_merge) or
        "p2p" (the attention kernel publishes its rows into every rank's
        receive area over peer memory; one merge kernel per rank).
        strict (p2p): check the merge's timeout status after every step (one
        host sync per step); with strict=False call check_exchange() yourself."""
        from .kv_cache import KvCache, lse_merge

        td = _dist()
        self.group = group
        self.world = td.get_world_size(group) if td.is_initialized() else 1
        self.rank = td.get_rank(group) if td.is_initialized() else 0
        self.B, self.Hq = batch, q_heads
        self.cache = KvCache(cfg, batch=batch, q_heads=q_heads, max_tokens=max_tokens_per_rank, device=device,
                             keep_exact=keep_exact)
        self.shard = None
        self._merge = merge or (lambda outs, lses: lse_merge(outs, lses))
        if exchange not in ("nccl", "p2p"):
            raise ValueError(f"exchange must be 'nccl' or 'p2p', not {exchange!r}")
        self.exchange = exchange
        self.peers = PeerExchange(batch * q_heads, device, group) if exchange == "p2p" and self.world > 1 else None
        self.strict = strict
        self._status = None
        self._ext = {}

    def _on(self, stream):
        """Run torch ops (gather, merge, fills) on the caller's stream, so they
        are ordered after the attention kernel launched there (and the reused
        result buffers are stream-ordered across steps)."""
        import torch

        if stream is None:
            return contextlib.nullcontext()
        s = self._ext.get(stream)
        if s is None:
            s = self._ext[stream] = torch.cuda.ExternalStream(stream, device=torch.device("cuda", self.cache.device))
        return torch.cuda.stream(s)

    def prefill(self, k, v, S: int | None = None, sliced: bool = False, stream=None):
        S = k.shape[1] if S is None else S
        self.shard = sequence_shard(S, self.world, self.rank)
        if not sliced:
            k = k[:, self.shard.tok_lo:self.shard.tok_hi].contiguous()
            v = v[:, self.shard.tok_lo:self.shard.tok_hi].contiguous()
        self.cache.buffer_quant(k, v, stream=stream)

    def local_partial(self, q, k=None, v=None, stream=None):
        """(O [B*Hq, d], LSE [B*Hq]) of this rank's shard; the tail rank also
        attends the current token and appends it (decode_step ordering)."""
        import torch

        rows = self.B * self.Hq
        if getattr(self, "_bufs", None) is None or self._bufs[0].device != q.device:
            self._bufs = (torch.empty((rows, D), dtype=torch.float32, device=q.device),
                          torch.empty((rows,), dtype=torch.float32, device=q.device))
        out, lse = self._bufs  # reused across steps (stream-ordered)
        if self.shard is not None and self.shard.tail and k is not None:
            self.cache.decode_step(q, k, v, out=out, lse=lse, stream=stream)
        elif self.cache.total_tokens > 0:
            self.cache.attend(q, out=out, lse=lse, stream=stream)
        else:  # an empty shard contributes nothing to the softmax
            out.zero_()
            lse.fill_(float("-inf"))
        return out, lse

    def decode_step(self, q, k, v, stream=None):
        with self._on(stream):  # every launch and torch op below on one stream
            if self.peers is not None:
                return self._decode_step_p2p(q, k, v)
            o, l = self.local_partial(q, k, v)
            if self.world == 1:  # the only shard: its partial is the normalised result
                return o.reshape(self.B, self.Hq, D)
            outs, lses = gather_partials(o, l, self.group)
            return self._merge(outs, lses).reshape(self.B, self.Hq, D)

    def _decode_step_p2p(self, q, k, v):
        import torch

        from . import kv_cache as kc

        px = self.peers
        px.epoch += 1
        if self.shard is not None and self.shard.tail and k is not None:
            self.cache.attend_publish(q, px.plan, px.epoch, k, v)
        elif self.cache.total_tokens > 0:
            self.cache.attend_publish(q, px.plan, px.epoch)
        else:
            kc.peer_publish_empty(px.plan, px.epoch)
        if getattr(self, "_p2p_out", None) is None:
            self._p2p_out = torch.empty((self.B * self.Hq, D), dtype=torch.float32, device=q.device)
            self._status = torch.zeros(1, dtype=torch.int32, device=q.device)
        kc.peer_merge(px.plan, px.epoch, self._p2p_out, status=self._status)
        if self.strict:
            self.check_exchange()
        return self._p2p_out.reshape(self.B, self.Hq, D)

    def check_exchange(self):
        """Raise if a peer-merge since the last check timed out (a rank did not
        publish within ~5 s; its rows were returned as NaN).  Synchronises."""
        if self._status is not None and int(self._status.item()) != 0:
            self._status.zero_()
            raise RuntimeError("sequence-shard exchange: a peer did not publish its (O, LSE) rows within 5 s")

    @property
    def total_tokens(self) -> int:
        import torch

        td = _dist()
        if self.world == 1:
            return self.cache.total_tokens
        t = torch.tensor([self.cache.total_tokens], dtype=torch.int64)
        if td.get_backend(self.group) == "nccl":
            t = t.cuda()
        td.all_reduce(t, group=self.group)
        return int(t.item())

    def close(self):
        if self.peers is not None:
            self.peers.close()
            self.peers = None
        self.cache.close()
