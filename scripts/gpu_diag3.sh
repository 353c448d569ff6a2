#!/bin/bash
export PYTHONUNBUFFERED=1
OUT=gpurun_out/d3; mkdir -p $OUT
for w in 8 4; do timeout 300 python scripts/diag_c5proxy.py $w 2>&1 | tail -1; done > $OUT/c5proxy.txt
export OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so
for spec in "8192 1 2 28 4" "131072 8 2 4 1" "32768 16 2 32 8"; do
  echo "=== $spec" ; timeout 300 python scripts/diag_timeline.py $spec 2>&1 | grep -v "^---" | tail -5
done > $OUT/timelines.txt 2>&1
