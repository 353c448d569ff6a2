"""Decode step with L2-hot vs HBM-cold per-step inputs (C2 INT2), back to back."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
B, S, Hq, Hkv = 16, 32768, 32, 8
dev = torch.device("cuda")
st = torch.cuda.Stream(); torch.cuda.set_stream(st); sh = st.cuda_stream
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 1024, keep_exact=False)
k, v = synth_kv(B, S, Hkv, 1, dev); cache.buffer_quant(k, v, stream=sh); del k, v
q, kn, vn = step_inputs(600, B, Hq, Hkv, 3, dev)
out = torch.empty((B, Hq, 128), device=dev)
def run(hot, n=100, base=0):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(n):
        j = 0 if hot else base + i
        cache.decode_step(q[j], kn[j], vn[j], out=out, stream=sh)
    e1.record(st); torch.cuda.synchronize()
    return round(1e3 * e0.elapsed_time(e1) / n, 2)
run(True, 20)
res = {"cold": run(False, 100, 100), "hot": run(True, 100), "cold2": run(False, 100, 300), "hot2": run(True, 100)}
print(json.dumps(res))
