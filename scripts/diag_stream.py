"""C5 streaming append (32 x 2048-token chunks, 4 KV heads) timed twice in one process."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
dev = torch.device("cuda"); H = 4
res = []
for rep in range(3):
    c = KvCache(PipelineConfig(heads=H, bits=2), batch=1, q_heads=28, max_tokens=256 + 32 * 2048, keep_exact=False)
    ka, va = synth_kv(1, 32 * 2048 + 100, H, 99, dev)
    c.buffer_quant(ka[:, :100].contiguous(), va[:, :100].contiguous())
    ch = [(ka[:, 100 + i * 2048:100 + (i + 1) * 2048].contiguous(), va[:, 100 + i * 2048:100 + (i + 1) * 2048].contiguous()) for i in range(32)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k_, v_ in ch: c.buffer_quant(k_, v_)
    e1.record(); torch.cuda.synchronize()
    res.append(round(e0.elapsed_time(e1), 3)); print(c.status()); c.close()
print(json.dumps({"ms": res}))
