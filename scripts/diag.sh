#!/bin/bash
# quick kernel-timing diagnostics (graph-timed attend, decode vs attend)
mkdir -p gpurun_out
for b in 2 4 0; do timeout 120 python scripts/sweep.py $b 2>&1 | tail -1; done | tee gpurun_out/diag_sweep.txt
timeout 120 python scripts/decode_vs_attend.py 2>&1 | tail -2 | tee gpurun_out/diag_dva.txt
timeout 600 python -m pytest tests/test_gpu_sharding.py -q -x 2>&1 | tail -15 | tee gpurun_out/diag_shard.txt
