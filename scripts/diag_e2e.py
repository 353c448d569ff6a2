"""Where does the host-buffer decode step spend its time? (C2 INT2)"""
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
t("host_api", lambda i: cache.decode_step_host(qn[i], kn_[i], vn_[i], on, stream=sh))
t("host_api_default_stream_lookup", lambda i: cache.decode_step_host(qn[i], kn_[i], vn_[i], on))
import ctypes
from paper_2605_19660_b200.kv_cache import lib
L = lib()
qp = [qn[i].ctypes.data for i in range(K)]; kp = [kn_[i].ctypes.data for i in range(K)]; vp = [vn_[i].ctypes.data for i in range(K)]
op = on.ctypes.data
t("raw_cabi", lambda i: L.oscar_kv_decode_step_host(cache._h, qp[i], kp[i], vp[i], op, None, sh))
qd = torch.empty((B, Hq, 128), dtype=torch.bfloat16, device=dev); kd = torch.empty((B, Hkv, 128), dtype=torch.bfloat16, device=dev)
vd = torch.empty_like(kd); od = torch.empty((B, Hq, 128), device=dev)
t("device_api_sync", lambda i: (cache.decode_step(qd, kd, vd, out=od, stream=sh), torch.cuda.current_stream().synchronize()))
def copies(i):
    qd.copy_(q_host[i], non_blocking=True); kd.copy_(k_host[i], non_blocking=True); vd.copy_(v_host[i], non_blocking=True)
    out_host.copy_(od, non_blocking=True); torch.cuda.current_stream().synchronize()
t("copies_only_sync", copies)
t("empty_sync", lambda i: torch.cuda.current_stream().synchronize())
print(json.dumps(res))
