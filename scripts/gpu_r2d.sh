#!/bin/bash
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 300 python scripts/diag_host.py 2>&1 | tail -1 | tee gpurun_out/diag_host.txt
for cfg in "32768 16" "8192 16" "131072 8"; do set -- $cfg
  OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so timeout 200 python scripts/diag_timeline.py $1 $2 2 2>&1 | grep -E "^---|timeline|end phases" | tail -3; done | tee gpurun_out/timeline.txt
