"""Prefill quantize time (bench.py's prefill leg: 16 x 32K x 8 heads, INT2/INT4 with the
fp64 shadow) and a 2048-token streaming append; device time, median of 5."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
dev = torch.device("cuda")
B, S, H = 16, 32768, 8
k, v = synth_kv(B, S, H, 1, dev)
res = {}
for bits in (2, 4):
    ts = []
    for r in range(5):
        c = KvCache(PipelineConfig(heads=H, bits=bits), batch=B, q_heads=32, max_tokens=S + 256)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c.buffer_quant(k, v); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1)); c.close()
    ts.sort(); res[f"prefill_int{bits}_ms"] = round(ts[2], 3)
ka, va = synth_kv(1, 2048 * 9 + 100, 4, 3, dev)
c = KvCache(PipelineConfig(heads=4, bits=2), batch=1, q_heads=28, max_tokens=2048 * 10 + 512, keep_exact=False)
c.buffer_quant(ka[:, :100].contiguous(), va[:, :100].contiguous())
ch = [(ka[:, 100 + i * 2048:100 + (i + 1) * 2048].contiguous(), va[:, 100 + i * 2048:100 + (i + 1) * 2048].contiguous()) for i in range(9)]
c.buffer_quant(*ch[0]); torch.cuda.synchronize()
ts = []
for i in range(1, 9):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c.buffer_quant(*ch[i]); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort(); res["append_2048_us"] = round(1e3 * ts[len(ts) // 2], 1)
print(json.dumps(res))
