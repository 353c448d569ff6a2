#!/bin/bash
# prefill quantize A/B (working tree vs HEAD build): GPU tests, prefill + streaming-append times, ncu of the prefill kernel
export PYTHONUNBUFFERED=1
OUT=${OUT:-gpurun_out/qab}; mkdir -p $OUT
H=$PWD/paper_2605_19660_b200/liboscar_b200_head.so; N=$PWD/paper_2605_19660_b200/liboscar_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for r in 1 2; do for v in head new; do L=$N; [ $v = head ] && L=$H
  echo "$v $(OSCAR_LIB=$L timeout 300 python scripts/diag_prefill.py 2>/dev/null | tail -1)"
done; done > $OUT/ab.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize_kernel -s 4 -c 1 \
  -o $OUT/prof_quant_int2 -f python bench.py --steps 2 --warmup 1 --no-compare --no-cpu > $OUT/ncu_quant.log 2>&1
# small-launch grid aligned to the segment count vs HEAD
[ -n "$SKIP_GRID" ] || for r in 1 2; do for v in head new; do L=$N; [ $v = head ] && L=$H
  for b in 8 4 2 1; do echo "$v c3_b$b $(OSCAR_LIB=$L timeout 300 python bench.py --config c3 --batch $b --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1), round(d["roofline"]["frac"],3))')"; done
  echo "$v c5_proxy8 $(OSCAR_LIB=$L timeout 300 python bench.py --config c5 --proxy-world 8 --steps 32 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"
  echo "$v C2 $(OSCAR_LIB=$L timeout 200 python bench.py --steps 128 --warmup 8 --no-compare --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["us_per_step"],2), round(d["e2e"]["us_per_step"],1), round(d["prefill_quantize"]["ms"],3))')"
done; done > $OUT/ab_grid.txt 2>&1
