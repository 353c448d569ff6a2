"""Where does the host-buffer decode step spend its time? (C2 INT2)
Whole-step wall time of several forms of the step, and -- for the split form
(copies + device entry + sync) -- device-side event times of the copies and the
kernel plus the host submission time."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
B, S, Hq, Hkv = 16, 32768, 32, 8
dev = torch.device("cuda")
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); sh = stream.cuda_stream
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 2048, keep_exact=False)
k, v = synth_kv(B, S, Hkv, 1, dev); cache.buffer_quant(k, v); del k, v
K = 100
qh, kh, vh = step_inputs(K, B, Hq, Hkv, 7, dev)
q_host = qh.cpu().pin_memory(); k_host = kh.cpu().pin_memory(); v_host = vh.cpu().pin_memory()
out_host = torch.empty((B, Hq, 128), dtype=torch.float32).pin_memory()
qn = q_host.view(torch.int16).numpy().view(np.uint16); kn_ = k_host.view(torch.int16).numpy().view(np.uint16)
vn_ = v_host.view(torch.int16).numpy().view(np.uint16); on = out_host.numpy()
res = {}
def t(name, fn, n=K):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for i in range(n): fn(i)
    torch.cuda.synchronize(); res[name] = round(1e6 * (time.perf_counter() - t0) / n, 1)
import ctypes
from paper_2605_19660_b200.kv_cache import lib
L = lib()
qp = [qn[i].ctypes.data for i in range(K)]; kp = [kn_[i].ctypes.data for i in range(K)]; vp = [vn_[i].ctypes.data for i in range(K)]
op = on.ctypes.data
t("raw_cabi_host_entry", lambda i: L.oscar_kv_decode_step_host(cache._h, qp[i], kp[i], vp[i], op, None, sh))
qd = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device=dev); kd = torch.empty((B, Hkv, 128), dtype=torch.bfloat16, device=dev)
vd = torch.empty_like(kd); od = torch.empty((B, Hq, 128), device=dev)
t("device_entry_sync", lambda i: (cache.decode_step(qd, kd, vd, out=od, stream=sh), stream.synchronize()))
t("device_entry_no_sync", lambda i: cache.decode_step(qd, kd, vd, out=od, stream=sh))
def copies(i):
    qd.copy_(q_host[i], non_blocking=True); kd.copy_(k_host[i], non_blocking=True); vd.copy_(v_host[i], non_blocking=True)
    out_host.copy_(od, non_blocking=True); stream.synchronize()
t("copies_only_sync", copies)
t("empty_sync", lambda i: stream.synchronize())
# split form with events: [copies] [kernel] [D2H], host submit time
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
acc = {"h2d": 0.0, "kernel": 0.0, "d2h": 0.0, "submit": 0.0, "wall": 0.0}
n = 50
for i in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record(stream)
    qd.copy_(q_host[i], non_blocking=True); kd.copy_(k_host[i], non_blocking=True); vd.copy_(v_host[i], non_blocking=True)
    ev[1].record(stream)
    cache.decode_step(qd, kd, vd, out=od, stream=sh)
    ev[2].record(stream)
    out_host.copy_(od, non_blocking=True)
    ev[3].record(stream)
    t1 = time.perf_counter()
    stream.synchronize()
    t2 = time.perf_counter()
    acc["h2d"] += ev[0].elapsed_time(ev[1]) * 1e3; acc["kernel"] += ev[1].elapsed_time(ev[2]) * 1e3
    acc["d2h"] += ev[2].elapsed_time(ev[3]) * 1e3; acc["submit"] += (t1 - t0) * 1e6; acc["wall"] += (t2 - t0) * 1e6
res["split_form_us"] = {k: round(v / n, 1) for k, v in acc.items()}
print(json.dumps(res))
