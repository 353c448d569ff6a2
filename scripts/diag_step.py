"""Why is a bench decode step slower than an attend?  Variants at C2 INT2."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig

B, S, Hq, Hkv, R = 16, 32768, 32, 8, 128
dev = torch.device("cuda")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
sh = stream.cuda_stream
keep = bool(int(os.environ.get("KEEP", "1")))
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 2048, keep_exact=keep)
k, v = synth_kv(B, S, Hkv, 1234, dev)
cache.buffer_quant(k, v)
del k, v
N = 128
q, kn, vn = step_inputs(8 * N, B, Hq, Hkv, 99, dev)
out = torch.empty((B, Hq, 128), device=dev)
lse = torch.empty((B, Hq), device=dev)
pos = [0]


def run(kind, per_step):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for i in range(N):
        if per_step:
            evs[i][0].record(stream)
        j = pos[0]
        if kind == "decode":
            cache.decode_step(q[j], kn[j], vn[j], out=out, stream=sh)
            pos[0] += 1
        else:
            cache.attend(q[j], out=out, lse=lse, stream=sh)
        if per_step:
            evs[i][1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    tot = 1e3 * e0.elapsed_time(e1) / N
    per = [1e3 * a.elapsed_time(b) for a, b in evs] if per_step else []
    return {"total_us": round(tot, 2), "per_step_avg_us": round(sum(per) / len(per), 2) if per else None,
            "per_step_min_us": round(min(per), 2) if per else None, "per_step_max_us": round(max(per), 2) if per else None}


res = {"keep_exact": keep}
res["decode_events"] = run("decode", True)
res["decode_noevents"] = run("decode", False)
res["attend_events"] = run("attend", True)
res["attend_noevents"] = run("attend", False)
t_end = time.time() + 0.4
while time.time() < t_end:
    for _ in range(20):
        cache.attend(q[0], out=out, lse=lse, stream=sh)
    torch.cuda.synchronize()
res["after_soak_decode_events"] = run("decode", True)
res["after_soak_attend_noevents"] = run("attend", False)
print(json.dumps(res))

# flush-step cost over several windows
flush_t = []
for rep in range(3):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(N)]
    r_before = []
    for i in range(N):
        r_before.append(cache.residual_tokens)
        evs[i][0].record(stream)
        j = pos[0]
        cache.decode_step(q[j], kn[j], vn[j], out=out, stream=sh)
        pos[0] += 1
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    per = [1e3 * a.elapsed_time(b) for a, b in evs]
    fl = [i for i in range(N) if r_before[i] == R - 1]
    flush_t.append([round(per[i], 1) for i in fl])
print(json.dumps({"flush_step_us": flush_t}))
