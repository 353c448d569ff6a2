"""Small end-to-end workload for compute-sanitizer: prefill (+ partial window),
decode steps across a flush, attend, host entry, multi-cache entry, LSE merge,
for INT2 / INT4 / bf16 and the explicit-V mode.  usage: python scripts/sanitize_all.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2605_19660_b200 import DecodeBatch, KvCache, PipelineConfig, lse_merge

torch.manual_seed(0)
B, H, g, S = 2, 2, 4, 8 * 128 + 100  # 8 packed blocks + 100-token window
for bits, rotv in ((2, False), (4, False), (0, False), (2, True)):
    k = torch.randn((B, S + 40, H, 128), device="cuda").to(torch.bfloat16)
    v = torch.randn((B, S + 40, H, 128), device="cuda").to(torch.bfloat16)
    q = torch.randn((B, H * g, 128), device="cuda").to(torch.bfloat16)
    c = KvCache(PipelineConfig(heads=H, bits=bits, rotate_v=rotv), batch=B, q_heads=H * g, max_tokens=S + 64)
    c.buffer_quant(k[:, :S].contiguous(), v[:, :S].contiguous())
    for t in range(S, S + 32):  # the 28th step fills the window: flush after attention
        c.decode_step(q, k[:, t].contiguous(), v[:, t].contiguous())
    o, l = c.attend(q)
    c.buffer_quant(k[:, S + 32:S + 34].contiguous(), v[:, S + 32:S + 34].contiguous())  # ring append
    qh = q.view(torch.int16).cpu().numpy().view(np.uint16)
    kh = k[:, S + 34].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    vh = v[:, S + 34].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    oh = np.zeros((B, H * g, 128), np.float32)
    c.decode_step_host(qh, kh, vh, oh)
    c2 = KvCache(PipelineConfig(heads=H, bits=bits, rotate_v=rotv), batch=B, q_heads=H * g, max_tokens=S + 64)
    c2.buffer_quant(k[:, :S].contiguous(), v[:, :S].contiguous())
    outs = [torch.empty((B, H * g, 128), device="cuda") for _ in range(2)]
    DecodeBatch([c, c2], [q, q], [k[:, S + 35].contiguous()] * 2, [v[:, S + 35].contiguous()] * 2, outs).run()
    m = lse_merge(torch.stack([o.reshape(-1, 128), o.reshape(-1, 128)]), torch.stack([l.reshape(-1), l.reshape(-1)]))
    torch.cuda.synchronize()
    print("ok", bits, rotv, float(m.abs().max()), c.flush_count)

# split-KV segments with more than 9 CTA partials (the ticket merge form): one sequence,
# one KV head, 80 blocks over ~10 CTAs
k = torch.randn((1, 80 * 128 + 4, 1, 128), device="cuda").to(torch.bfloat16)
v = torch.randn((1, 80 * 128 + 4, 1, 128), device="cuda").to(torch.bfloat16)
q = torch.randn((1, 4, 128), device="cuda").to(torch.bfloat16)
c = KvCache(PipelineConfig(heads=1, bits=2), batch=1, q_heads=4, max_tokens=80 * 128 + 64)
c.buffer_quant(k[:, :80 * 128].contiguous(), v[:, :80 * 128].contiguous())
for t in range(80 * 128, 80 * 128 + 2):
    c.decode_step(q, k[:, t].contiguous(), v[:, t].contiguous())
# host entry with page-locked buffers: the kernel reads q/k/v and writes out over PCIe
qp = q.cpu().pin_memory().view(torch.int16).numpy().view(np.uint16)
kp = k[:, 80 * 128 + 2].contiguous().cpu().pin_memory().view(torch.int16).numpy().view(np.uint16)
vp = v[:, 80 * 128 + 2].contiguous().cpu().pin_memory().view(torch.int16).numpy().view(np.uint16)
op = torch.zeros((1, 4, 128), dtype=torch.float32).pin_memory().numpy()
c.decode_step_host(qp, kp, vp, op)
torch.cuda.synchronize()
print("ok ticket-form + pinned host entry", float(np.abs(op).max()), c.status())
# fused sequence-shard exchange: 2 virtual ranks, 2 epochs
from paper_2605_19660_b200 import kv_cache as kcm
from paper_2605_19660_b200.sharding import local_peer_plans
plans, areas = local_peer_plans(2, 4)
shards = []
for r in range(2):
    cs = KvCache(PipelineConfig(heads=1, bits=2), batch=1, q_heads=4, max_tokens=4 * 128 + 64)
    cs.buffer_quant(k[:, r * 512:(r + 1) * 512].contiguous(), v[:, r * 512:(r + 1) * 512].contiguous())
    shards.append(cs)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for ep in (1, 2):
    for r in range(2):
        shards[r].attend_publish(q, plans[r], ep)
    outs = [torch.empty((4, 128), device="cuda") for _ in range(2)]
    for r in range(2):
        kcm.peer_merge(plans[r], ep, outs[r], status=st)
torch.cuda.synchronize()
print("ok peer exchange", int(st.item()), float((outs[0] - outs[1]).abs().max()))
