#!/bin/bash
# TILES kernel (window tiles as ring units) for small launches vs HEAD
export PYTHONUNBUFFERED=1
OUT=gpurun_out/tiles3; mkdir -p $OUT
H=$PWD/paper_2605_19660_b200/liboscar_b200_head.so; N=$PWD/paper_2605_19660_b200/liboscar_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
OSCAR_TILE_UNITS=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py tests/test_gpu_scale.py tests/test_gpu_numerics.py -q -x > $OUT/pytest_forced.txt 2>&1; echo "rc=$?" >> $OUT/pytest_forced.txt
for r in 1 2; do for v in head new; do L=$N; [ $v = head ] && L=$H
  echo "$v C2 $(OSCAR_LIB=$L timeout 200 python bench.py --steps 128 --warmup 8 --no-compare --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["us_per_step"],2), round(d["e2e"]["us_per_step"],1))')"
done; done > $OUT/ab.txt 2>&1
for v in head new; do L=$N; [ $v = head ] && L=$H
  for b in 64 8 1; do echo "$v c3_b$b $(OSCAR_LIB=$L timeout 300 python bench.py --config c3 --batch $b --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1), round(d["roofline"]["frac"],3))')"; done
  for c in c5 c4; do echo "$v ${c}_proxy8 $(OSCAR_LIB=$L timeout 300 python bench.py --config $c --proxy-world 8 --steps 32 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1), round(d["roofline"]["frac"],3))')"; done
done >> $OUT/ab.txt 2>&1
