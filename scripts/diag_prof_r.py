"""OSCAR_PROF phase breakdown + per-CTA dump of attend at residual fill r (C2 INT2).
usage: OSCAR_PROF=1 OSCAR_PROF_FILE=... OSCAR_LIB=.../liboscar_b200_prof.so python scripts/diag_prof_r.py r
(profiling library: make -C paper_2605_19660_b200/csrc PROF=1)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
r = int(sys.argv[1])
B, S, Hq, Hkv = 16, 32768, 32, 8
dev = torch.device("cuda")
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 256, keep_exact=False)
k, v = synth_kv(B, S, Hkv, 1, dev); cache.buffer_quant(k, v); del k, v
q, kn, vn = step_inputs(200, B, Hq, Hkv, 3, dev)
out = torch.empty((B, Hq, 128), device=dev); lse = torch.empty((B, Hq), device=dev)

step = 0
while cache.residual_tokens < r:
    cache.decode_step(q[step], kn[step], vn[step], out=out); step += 1
torch.cuda.synchronize()
cache.attend(q[0], out, lse)
torch.cuda.synchronize()
