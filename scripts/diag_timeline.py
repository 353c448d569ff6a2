"""Per-launch timeline of one attend (globaltimer stamps of the profiling build):
entry spread, end of streaming per warp, exit.  C2 shape by default.
usage: OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so \
       python scripts/diag_timeline.py [ctx] [batch] [bits] [q heads] [kv heads]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig

ctx = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
bits = int(sys.argv[3]) if len(sys.argv) > 3 else 2
Hq = int(sys.argv[4]) if len(sys.argv) > 4 else 32
Hkv = int(sys.argv[5]) if len(sys.argv) > 5 else 8
dev = torch.device("cuda")
cache = KvCache(PipelineConfig(heads=Hkv, bits=bits), batch=B, q_heads=Hq, max_tokens=ctx + 256, keep_exact=False)
k, v = synth_kv(B, ctx, Hkv, 1, dev)
cache.buffer_quant(k, v)
del k, v
q = torch.randn((B, Hq, 128), device=dev).to(torch.bfloat16)
out = torch.empty((B, Hq, 128), device=dev)
lse = torch.empty((B, Hq), device=dev)
for i in range(3):
    print(f"--- ctx {ctx} B {B} bits {bits} launch {i}", file=sys.stderr, flush=True)
    cache.attend(q, out, lse)
    torch.cuda.synchronize()
