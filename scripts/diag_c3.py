"""C3 per-layer costs at small batch: attend vs decode_step (one cache, back to back)
and a 32-layer decode_step_many, device time per layer.  usage: python scripts/diag_c3.py B"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import DecodeBatch, KvCache, PipelineConfig
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
S, Hq, Hkv, L = 8192, 28, 4, 32
dev = torch.device("cuda")
st = torch.cuda.Stream(); torch.cuda.set_stream(st); sh = st.cuda_stream
caches = []
for l in range(L):
    c = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 512, keep_exact=False)
    k, v = synth_kv(B, S, Hkv, 7 + l, dev); c.buffer_quant(k, v, stream=sh); del k, v
    caches.append(c)
q, kn, vn = step_inputs(300, B, Hq, Hkv, 11, dev)
out = torch.empty((B, Hq, 128), device=dev); lse = torch.empty((B, Hq), device=dev)
torch.cuda.synchronize()
def timeit(fn, n):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(n): fn(i)
    e1.record(st); torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / n
res = {"B": B}
res["attend_us"] = timeit(lambda i: caches[0].attend(q[0], out, lse, stream=sh), 50)
pos = [0]
def dec(i):
    caches[1].decode_step(q[pos[0]], kn[pos[0]], vn[pos[0]], out=out, stream=sh); pos[0] += 1
res["decode_us"] = timeit(dec, 50)
def many(i):
    j = 100 + i
    DecodeBatch(caches, [q[j]] * L, [kn[j]] * L, [vn[j]] * L, [out] * L).run(sh)
res["many_per_layer_us"] = timeit(many, 10) / L
def attend_all(i):
    for c in caches: c.attend(q[0], out, lse, stream=sh)
res["attend_32_per_layer_us"] = timeit(attend_all, 10) / L
print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in res.items()}))
# device time of the 32 attends with no host gaps: one CUDA graph
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    for c in caches: c.attend(q[0], out, lse, stream=sh)
torch.cuda.synchronize()
res["attend_32_graph_per_layer_us"] = timeit(lambda i: g.replay(), 20) / L
# host submission cost of one decode_step_many call (no device wait)
import time
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(5):
    j = 200 + i
    DecodeBatch(caches, [q[j]] * L, [kn[j]] * L, [vn[j]] * L, [out] * L).run(sh)
res["many_host_per_layer_us"] = 1e6 * (time.perf_counter() - t0) / 5 / L
torch.cuda.synchronize()
print(json.dumps({k: round(v, 2) if isinstance(v, float) else v for k, v in res.items()}))
