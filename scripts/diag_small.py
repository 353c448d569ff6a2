"""Latency of small decode-attention launches (C3 per-layer shapes): graph-timed attend + phase profile.
usage: python scripts/diag_small.py B S [Hkv Hq]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
B, S = int(sys.argv[1]), int(sys.argv[2])
Hkv = int(sys.argv[3]) if len(sys.argv) > 3 else 4
Hq = int(sys.argv[4]) if len(sys.argv) > 4 else 28
dev = torch.device("cuda")
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 256, keep_exact=False)
k, v = synth_kv(B, S, Hkv, 1, dev); cache.buffer_quant(k, v); del k, v
q = torch.randn((B, Hq, 128), device=dev).to(torch.bfloat16)
out = torch.empty((B, Hq, 128), device=dev); lse = torch.empty((B, Hq), device=dev)
for _ in range(10): cache.attend(q, out, lse)
torch.cuda.synchronize()
n = 50
s_cap = torch.cuda.Stream(); s_cap.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s_cap):
    with torch.cuda.graph(g, stream=s_cap):
        for _ in range(n): cache.attend(q, out, lse)
torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3): g.replay()
e1.record(); torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / (3 * n)
byt = B * Hkv * (S // 128) * 12800
print(json.dumps({"B": B, "S": S, "Hkv": Hkv, "Hq": Hq, "graph_us": round(us, 2), "GBps": round(byt / us / 1e3, 1)}))
