"""Kernel-config sweep: attend-only latency at the C2 workload (B=16, 32K, 32/8 heads).
usage: OSCAR_NCW=.. python scripts/sweep.py BITS"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import BLOCK_BYTES, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig

bits = int(sys.argv[1])
B, S, Hq, Hkv = 16, 32768, 32, 8
ctx = int(os.environ.get("SWEEP_CTX", S))
cache = KvCache(PipelineConfig(heads=Hkv, bits=bits), batch=B, q_heads=Hq, max_tokens=ctx + 64, keep_exact=False)
k, v = synth_kv(B, ctx, Hkv, 1, torch.device("cuda"))
cache.buffer_quant(k, v)
del k, v
q = torch.randn((B, Hq, 128), device="cuda").to(torch.bfloat16)
out = torch.empty((B, Hq, 128), device="cuda")
lse = torch.empty((B, Hq), device="cuda")
for _ in range(10):
    cache.attend(q, out, lse)
torch.cuda.synchronize()
# CUDA-graph the launches so host overhead never shows up in the device timing
n = 20
s_cap = torch.cuda.Stream()
s_cap.wait_stream(torch.cuda.current_stream())
graph = torch.cuda.CUDAGraph()
with torch.cuda.stream(s_cap):
    with torch.cuda.graph(graph, stream=s_cap):
        for _ in range(n):
            cache.attend(q, out, lse)
torch.cuda.synchronize()
graph.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    graph.replay()
e1.record()
torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / (3 * n)
byt = B * Hkv * (ctx // 128) * BLOCK_BYTES[bits]
print(json.dumps({"bits": bits, "ncw": os.environ.get("OSCAR_NCW", "default"),
                  "ctx": ctx, "us": round(us, 2),
                  "GBps": round(byt / us / 1e3, 1)}))
