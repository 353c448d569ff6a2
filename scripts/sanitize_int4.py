"""Mid-size INT4/INT2 decode for compute-sanitizer (ring wraps: >NST units per CTA)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_19660_b200 import KvCache, PipelineConfig

bits = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B, S, H, g = 1, 32768, 8, 4
k = torch.randn((B, S, H, 128), device="cuda").to(torch.bfloat16)
v = torch.randn((B, S, H, 128), device="cuda").to(torch.bfloat16)
c = KvCache(PipelineConfig(heads=H, bits=bits), batch=B, q_heads=H * g, max_tokens=S + 16, keep_exact=False)
c.buffer_quant(k, v)
torch.cuda.synchronize()
q = torch.randn((B, H * g, 128), device="cuda").to(torch.bfloat16)
for i in range(3):
    out = c.decode_step(q, k[:, i].contiguous(), v[:, i].contiguous())
torch.cuda.synchronize()
print("ok", bits, float(out.abs().max()))
