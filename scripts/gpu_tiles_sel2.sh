#!/bin/bash
# TILES selection extended to 1.5-4 segments per CTA (TILES supersedes DEFER there) vs HEAD; + C5 / C3 B=8 timelines
export PYTHONUNBUFFERED=1
OUT=gpurun_out/tiles8; mkdir -p $OUT
H=$PWD/paper_2605_19660_b200/liboscar_b200_head.so; N=$PWD/paper_2605_19660_b200/liboscar_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for r in 1 2; do for v in head new; do L=$N; [ $v = head ] && L=$H
  for b in 256 192 160 128 64; do
  echo "$v c3_b$b $(OSCAR_LIB=$L timeout 300 python bench.py --config c3 --batch $b --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1), round(d["roofline"]["frac"],3))')"
  done
  echo "$v C2 $(OSCAR_LIB=$L timeout 200 python bench.py --steps 128 --warmup 8 --no-compare --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["us_per_step"],2), round(d["e2e"]["us_per_step"],1))')"
done; done > $OUT/ab.txt 2>&1
P=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so
for shape in "524288 1 2 28 4" "8192 8 2 28 4" "8192 1 2 28 4"; do
  echo "=== $shape" >> $OUT/timelines.txt
  OSCAR_PROF=1 OSCAR_LIB=$P timeout 300 python scripts/diag_timeline.py $shape >> $OUT/timelines.txt 2>&1
done
