"""Attend latency over a 3 s sustained run (power/clock behaviour) + nvidia-smi samples."""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
B, S, Hq, Hkv = 16, 32768, 32, 8
dev = torch.device("cuda")
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); sh = stream.cuda_stream
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 1024, keep_exact=False)
k, v = synth_kv(B, S, Hkv, 1234, dev); cache.buffer_quant(k, v); del k, v
q, kn, vn = step_inputs(4, B, Hq, Hkv, 99, dev)
out = torch.empty((B, Hq, 128), device=dev); lse = torch.empty((B, Hq), device=dev)
smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active",
                        "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
time.sleep(0.5)
res = []
t0 = time.time()
while time.time() - t0 < 3.0:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(50):
        cache.attend(q[0], out=out, lse=lse, stream=sh)
    e1.record(stream)
    torch.cuda.synchronize()
    res.append((round(time.time() - t0, 3), round(1e3 * e0.elapsed_time(e1) / 50, 2)))
time.sleep(1.0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(50):
    cache.attend(q[0], out=out, lse=lse, stream=sh)
e1.record(stream); torch.cuda.synchronize()
after_idle = round(1e3 * e0.elapsed_time(e1) / 50, 2)
smi.terminate()
lines = smi.stdout.read().strip().splitlines()
print(json.dumps({"trace": res[::max(1, len(res) // 30)], "after_1s_idle": after_idle, "smi": lines[::3]}))
