"""Prefill quantize time (oscar_kv_append of B x S x H, INT2) -- device time per call."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
B, S, H = 16, 32768, 8
bits = int(sys.argv[1]) if len(sys.argv) > 1 else 2
k, v = synth_kv(B, S, H, 1, torch.device("cuda"))
ts = []
for i in range(4):
    c = KvCache(PipelineConfig(heads=H, bits=bits), batch=B, q_heads=32, max_tokens=S + 256, keep_exact=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c.buffer_quant(k, v); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1)); c.close()
print(json.dumps({"gpar": os.environ.get("OSCAR_QGPAR", "1"), "bits": bits, "ms": [round(t, 3) for t in ts]}))
