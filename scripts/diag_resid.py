"""Attention latency vs residual-window fill r, eager vs CUDA-graph timed (C2 INT2 by
default; DIAG_SHAPE=c3b1|c3b8|c3b64|c3b256 for one C3 layer at that batch).
usage: python scripts/diag_resid.py [bits]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 2
B, S, Hq, Hkv = {"c2": (16, 32768, 32, 8), "c3b1": (1, 8192, 28, 4), "c3b8": (8, 8192, 28, 4),
                 "c3b64": (64, 8192, 28, 4), "c3b256": (256, 8192, 28, 4)}[os.environ.get("DIAG_SHAPE", "c2")]
dev = torch.device("cuda")
cache = KvCache(PipelineConfig(heads=Hkv, bits=bits), batch=B, q_heads=Hq, max_tokens=S + 256, keep_exact=False)
k, v = synth_kv(B, S, Hkv, 1, dev)
cache.buffer_quant(k, v)
del k, v
q, kn, vn = step_inputs(200, B, Hq, Hkv, 3, dev)
out = torch.empty((B, Hq, 128), device=dev)
lse = torch.empty((B, Hq), device=dev)


def eager(n=40):
    for _ in range(5):
        cache.attend(q[0], out, lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        cache.attend(q[0], out, lse)
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n


def graphed(n=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                cache.attend(q[0], out, lse)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / (3 * n)


res = {}
step = 0
for r in (0, 1, 32, 64, 127):
    while cache.residual_tokens < r:
        cache.decode_step(q[step], kn[step], vn[step], out=out)
        step += 1
    torch.cuda.synchronize()
    res[r] = {"eager_us": round(eager(), 2), "graph_us": round(graphed(), 2)}
print(json.dumps({"bits": bits, "by_residual": res}))
