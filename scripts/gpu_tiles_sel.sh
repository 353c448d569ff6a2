#!/bin/bash
# TILES selection (small launches + 1.5-2 segments per CTA + host-buffer entry) vs HEAD (small launches only)
export PYTHONUNBUFFERED=1
OUT=gpurun_out/tiles6; mkdir -p $OUT
H=$PWD/paper_2605_19660_b200/liboscar_b200_head.so; N=$PWD/paper_2605_19660_b200/liboscar_b200.so
[ -n "$SKIP_TESTS" ] || { timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt; }
[ -n "$SKIP_C2" ] || for r in 1 2 3; do for v in head new; do L=$N; [ $v = head ] && L=$H
  echo "$v C2 $(OSCAR_LIB=$L timeout 200 python bench.py --steps 128 --warmup 8 --no-compare --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["us_per_step"],2), round(d["e2e"]["us_per_step"],1))')"
done; done > $OUT/ab.txt 2>&1
for r in 1 2; do for v in head new; do L=$N; [ $v = head ] && L=$H
  echo "$v c3_b64 $(OSCAR_LIB=$L timeout 300 python bench.py --config c3 --batch 64 --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1), round(d["roofline"]["frac"],3))')"
  echo "$v c3_proxy4 $(OSCAR_LIB=$L timeout 300 python bench.py --config c3 --proxy-world 4 --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1))')"
  for c in c4 c5; do echo "$v ${c}_1gpu $(OSCAR_LIB=$L timeout 300 python bench.py --config $c --steps 64 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"; done
done; done >> $OUT/ab.txt 2>&1
