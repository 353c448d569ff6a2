#!/bin/bash
export PYTHONUNBUFFERED=1 OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so
mkdir -p gpurun_out
for cfg in "32768 16" "8192 16" "131072 8" ; do set -- $cfg
  timeout 200 python scripts/diag_timeline.py $1 $2 2 2>&1 | grep -E "^---|OSCAR_PROF" ; done | tee gpurun_out/timeline.txt
