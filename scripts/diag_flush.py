"""First-flush anomaly: host vs device time of the steps around the first flushes."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
B, S, Hq, Hkv, R = 16, 32768, 32, 8, 128
dev = torch.device("cuda")
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); sh = stream.cuda_stream
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 1024, keep_exact=True)
k, v = synth_kv(B, S, Hkv, 1234, dev); cache.buffer_quant(k, v); del k, v
q, kn, vn = step_inputs(400, B, Hq, Hkv, 99, dev)
out = torch.empty((B, Hq, 128), device=dev)
torch.cuda.synchronize()
rows = []
for i in range(300):
    r = cache.residual_tokens
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(stream)
    cache.decode_step(q[i], kn[i], vn[i], out=out, stream=sh)
    e1.record(stream); t1 = time.perf_counter()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    rows.append((i, r, round(1e6 * (t1 - t0), 1), round(1e3 * e0.elapsed_time(e1), 1), round(1e6 * (t2 - t0), 1)))
print(json.dumps([x for x in rows if x[1] in (126, 127, 0) or x[0] < 3]))
