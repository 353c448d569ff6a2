#!/bin/bash
# small-launch timelines (profiling build): C3 B=1 / B=8 layer, C4 rank shard of 8, C5 tail shard of 8
export PYTHONUNBUFFERED=1 OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so
OUT=gpurun_out/d2; mkdir -p $OUT
for spec in "8192 1 2 28 4" "8192 8 2 28 4" "131072 8 2 4 1" "65536 1 2 28 4" "524288 1 2 28 4" "32768 16 2 32 8"; do
  echo "=== $spec" ; timeout 300 python scripts/diag_timeline.py $spec 2>&1 | grep -v "^---" | tail -4
done > $OUT/timelines.txt 2>&1
unset OSCAR_PROF OSCAR_LIB
for n in 8 4; do
  timeout 600 python bench.py --config c5 --proxy-world $n --steps 32 --warmup 4 > $OUT/proxy_c5_$n.json 2> $OUT/proxy_c5_$n.err
done
ls -la $OUT
