"""OSCAR_PROF phase breakdown of one attend launch for a config shape.
usage: OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so python scripts/diag_prof_cfg.py B S Hq Hkv
(build the profiling library first: make -C paper_2605_19660_b200/csrc PROF=1)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import step_inputs, synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
B, S, Hq, Hkv = (int(x) for x in sys.argv[1:5])
dev = torch.device("cuda")
cache = KvCache(PipelineConfig(heads=Hkv, bits=2), batch=B, q_heads=Hq, max_tokens=S + 256, keep_exact=False)
k, v = synth_kv(B, S, Hkv, 1, dev); cache.buffer_quant(k, v); del k, v
q, kn, vn = step_inputs(4, B, Hq, Hkv, 3, dev)
out = torch.empty((B, Hq, 128), device=dev); lse = torch.empty((B, Hq), device=dev)
cache.decode_step(q[0], kn[0], vn[0], out=out)
torch.cuda.synchronize()
for _ in range(2):
    cache.attend(q[1], out, lse)
torch.cuda.synchronize()
