"""Host-side cost of the C-ABI entries at the C2 shape (B=16, 32K, INT2):
per-call submission time of oscar_kv_attend / oscar_kv_decode_step (device pointers,
no sync), cudaPointerGetAttributes, and the synchronous host-buffer entry.
usage: python scripts/diag_host.py"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
from paper_2605_19660_b200.kv_cache import lib

B, S, Hq, Hkv = 16, 32768, 32, 8
dev = torch.device("cuda")
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 4096, keep_exact=False)
k, v = synth_kv(B, S, Hkv, 1, dev)
cache.buffer_quant(k, v)
del k, v
q, kn, vn = step_inputs(4, B, Hq, Hkv, 3, dev)
out = torch.empty((B, Hq, 128), device=dev)
L = lib()
h = cache._h
stream = torch.cuda.Stream()
sh = stream.cuda_stream
res = {}

# (1) attend: host submission cost per call (the GPU falls behind; no sync inside)
n = 400
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    L.oscar_kv_attend(h, q[0].data_ptr(), out.data_ptr(), None, sh)
t1 = time.perf_counter()
torch.cuda.synchronize()
res["attend_submit_us"] = 1e6 * (t1 - t0) / n

# (2) decode_step submission (appends: 200 steps cross at most 2 flushes)
n = 200
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(n):
    L.oscar_kv_decode_step(h, q[i % 4].data_ptr(), kn[i % 4].data_ptr(), vn[i % 4].data_ptr(), out.data_ptr(), None, sh)
t1 = time.perf_counter()
torch.cuda.synchronize()
res["decode_submit_us"] = 1e6 * (t1 - t0) / n

# (3) cudaPointerGetAttributes through torch's runtime (same cost class as ours)
try:
    rt = ctypes.CDLL("libcudart.so.12")
    buf = ctypes.create_string_buffer(64)
    pin = torch.empty(1 << 20, dtype=torch.uint8).pin_memory()
    t0 = time.perf_counter()
    for _ in range(1000):
        rt.cudaPointerGetAttributes(buf, ctypes.c_void_p(pin.data_ptr()))
    res["pointer_attr_us"] = 1e3 * (time.perf_counter() - t0)
except OSError as e:
    res["pointer_attr_us"] = str(e)

# (4) host-buffer entry, synchronous per step
qh = q.cpu().pin_memory().view(torch.int16).numpy()
kh = kn.cpu().pin_memory().view(torch.int16).numpy()
vh = vn.cpu().pin_memory().view(torch.int16).numpy()
oh = torch.empty((B, Hq, 128), dtype=torch.float32).pin_memory().numpy()
n = 200
for i in range(10):
    L.oscar_kv_decode_step_host(h, qh[i % 4].ctypes.data, kh[i % 4].ctypes.data, vh[i % 4].ctypes.data, oh.ctypes.data, None, sh)
t0 = time.perf_counter()
for i in range(n):
    L.oscar_kv_decode_step_host(h, qh[i % 4].ctypes.data, kh[i % 4].ctypes.data, vh[i % 4].ctypes.data, oh.ctypes.data, None, sh)
res["host_entry_us"] = 1e6 * (time.perf_counter() - t0) / n

# (5) device entry + per-step stream sync (no copies): launch + completion latency
t0 = time.perf_counter()
for i in range(n):
    L.oscar_kv_decode_step(h, q[i % 4].data_ptr(), kn[i % 4].data_ptr(), vn[i % 4].data_ptr(), out.data_ptr(), None, sh)
    stream.synchronize()
res["device_entry_sync_us"] = 1e6 * (time.perf_counter() - t0) / n

# (6) device time of the same steps (events on the stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for i in range(n):
    L.oscar_kv_decode_step(h, q[i % 4].data_ptr(), kn[i % 4].data_ptr(), vn[i % 4].data_ptr(), out.data_ptr(), None, sh)
e1.record(stream)
torch.cuda.synchronize()
res["device_us"] = 1e3 * e0.elapsed_time(e1) / n
print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}))
