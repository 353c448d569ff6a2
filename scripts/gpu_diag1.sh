#!/bin/bash
# round-2 diagnostics: C2 timeline (profiling build), C3 small-batch host vs device,
# e2e breakdown, per-rank proxy lines
export PYTHONUNBUFFERED=1
OUT=gpurun_out/d1; mkdir -p $OUT
OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so timeout 300 python scripts/diag_timeline.py > $OUT/timeline_c2.txt 2>&1
for b in 1 8 64; do timeout 300 python scripts/diag_c3.py $b 2>&1 | tail -1; done > $OUT/c3.txt
timeout 300 python scripts/diag_e2e.py > $OUT/e2e.txt 2>&1
for n in 8 4 2; do
  timeout 600 python bench.py --config c3 --proxy-world $n --steps 16 --warmup 3 > $OUT/proxy_c3_$n.json 2> $OUT/proxy_c3_$n.err
  timeout 600 python bench.py --config c4 --proxy-world $n --steps 32 --warmup 4 > $OUT/proxy_c4_$n.json 2> $OUT/proxy_c4_$n.err
  timeout 600 python bench.py --config c5 --proxy-world $n --steps 32 --warmup 4 > $OUT/proxy_c5_$n.json 2> $OUT/proxy_c5_$n.err
done
ls -la $OUT
