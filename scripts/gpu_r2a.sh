#!/bin/bash
# round-2 diagnostics: host-side entry costs, context sweep (steady rate vs fixed
# cost), variant A/B
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python scripts/diag_host.py 2>&1 | tail -2 | tee gpurun_out/diag_host.txt
for ctx in 4096 8192 16384 32768 65536; do SWEEP_CTX=$ctx timeout 120 python scripts/sweep.py 2 | tail -1; done | tee gpurun_out/ctx_sweep.txt
bash scripts/variants.sh run base imad 2>&1 | tee gpurun_out/variants.txt
