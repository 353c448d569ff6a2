"""decode_step vs attend latency, back-to-back (no per-step host work besides the call)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig

B, S, Hq, Hkv = 16, 32768, 32, 8
dev = torch.device("cuda")
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 1024, keep_exact=True)
k, v = synth_kv(B, S, Hkv, 1, dev)
cache.buffer_quant(k, v)
del k, v
q, kn, vn = step_inputs(400, B, Hq, Hkv, 3, dev)
out = torch.empty((B, Hq, 128), device=dev)
lse = torch.empty((B, Hq), device=dev)
res = {}


def timeit(fn, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n, 1e6 * (t1 - t0) / n


res["attend_r0"] = timeit(lambda i: cache.attend(q[0], out, lse), 50)
res["decode_first100"] = timeit(lambda i: cache.decode_step(q[i], kn[i], vn[i], out=out), 100)  # r 0..99
res["attend_r100"] = timeit(lambda i: cache.attend(q[0], out, lse), 50)
res["decode_next100"] = timeit(lambda i: cache.decode_step(q[100 + i], kn[100 + i], vn[100 + i], out=out), 100)
print(json.dumps({k: [round(x, 2) for x in v] for k, v in res.items()}), "(device us/call, host us/call)")
