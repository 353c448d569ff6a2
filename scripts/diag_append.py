"""Streaming append (C5 tail rank: 2048-token chunks, 4 KV heads, INT2) for ncu: a warm-up
chunk, then 4 timed chunks; each chunk is one quantize_kernel launch (16 R-blocks x 4
heads, 4 groups per CTA in parallel) + one ring copy of the remainder."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
dev = torch.device("cuda")
ka, va = synth_kv(1, 2048 * 6 + 100, 4, 3, dev)
c = KvCache(PipelineConfig(heads=4, bits=2), batch=1, q_heads=28, max_tokens=2048 * 7 + 512, keep_exact=False)
c.buffer_quant(ka[:, :100].contiguous(), va[:, :100].contiguous())
ch = [(ka[:, 100 + i * 2048:100 + (i + 1) * 2048].contiguous(), va[:, 100 + i * 2048:100 + (i + 1) * 2048].contiguous())
      for i in range(6)]
ts = []
for i in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c.buffer_quant(*ch[i]); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(json.dumps({"append_2048_us": [round(1e3 * t, 1) for t in ts]}))
