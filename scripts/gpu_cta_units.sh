#!/bin/bash
# packed units per CTA of small launches (OSCAR_CTA_UNITS; default 8): grid size vs fan-in of the split-KV merge
export PYTHONUNBUFFERED=1
OUT=gpurun_out/ctau; mkdir -p $OUT
for r in 1 2; do for u in 8 16 24 32 48; do
  echo "u$u c5_proxy8 $(OSCAR_CTA_UNITS=$u timeout 300 python bench.py --config c5 --proxy-world 8 --steps 32 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"
  echo "u$u c5_proxy4 $(OSCAR_CTA_UNITS=$u timeout 300 python bench.py --config c5 --proxy-world 4 --steps 32 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"
  echo "u$u c3_b8 $(OSCAR_CTA_UNITS=$u timeout 300 python bench.py --config c3 --batch 8 --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1))')"
  echo "u$u c3_b1 $(OSCAR_CTA_UNITS=$u timeout 300 python bench.py --config c3 --batch 1 --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1))')"
  echo "u$u c4_proxy8 $(OSCAR_CTA_UNITS=$u timeout 300 python bench.py --config c4 --proxy-world 8 --steps 32 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"
done; done > $OUT/ab.txt 2>&1
# ticket-form final merge with 40 partials per batch (one round trip for C5's ~38) vs 32: OSK_TICKET_FB variant build
F=$PWD/paper_2605_19660_b200/liboscar_b200_fb40.so
for r in 1 2; do for v in base fb40; do L=$PWD/paper_2605_19660_b200/liboscar_b200.so; [ $v = fb40 ] && L=$F
  echo "$v c5_1gpu $(OSCAR_LIB=$L timeout 300 python bench.py --config c5 --steps 64 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"
  echo "$v c5_proxy8 $(OSCAR_LIB=$L timeout 300 python bench.py --config c5 --proxy-world 8 --steps 32 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"
  echo "$v C2 $(OSCAR_LIB=$L timeout 200 python bench.py --steps 128 --warmup 8 --no-compare --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["us_per_step"],2))')"
done; done >> $OUT/ab.txt 2>&1
