#!/bin/bash
export PYTHONUNBUFFERED=1 OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so
mkdir -p gpurun_out/cta
cat > /tmp/tl.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from bench import synth_kv
from paper_2605_19660_b200 import KvCache, PipelineConfig
ctx, B = 32768, 16
dev = torch.device("cuda")
cache = KvCache(PipelineConfig(heads=8, bits=2), batch=B, q_heads=32, max_tokens=ctx + 256, keep_exact=False)
k, v = synth_kv(B, ctx, 8, 1, dev); cache.buffer_quant(k, v); del k, v
q = torch.randn((B, 32, 128), device=dev).to(torch.bfloat16)
out = torch.empty((B, 32, 128), device=dev); lse = torch.empty((B, 32), device=dev)
for i in range(6):
    os.environ["OSCAR_PROF_FILE"] = f"gpurun_out/cta/c2_launch{i}.csv"
    cache.attend(q, out, lse); torch.cuda.synchronize()
PY
timeout 200 python /tmp/tl.py 2>&1 | grep timeline
