#!/bin/bash
# stream-K split weights: OSCAR_SEG_COST (per segment, default 3) / OSCAR_TAIL_COST (per residual tail, default 6)
export PYTHONUNBUFFERED=1
OUT=gpurun_out/segc; mkdir -p $OUT
for sc in 3 0 6 12; do for tc in 6 2 12; do
  [ $sc != 3 ] && [ $tc != 6 ] && continue
  echo "sc$sc tc$tc c3_b256 $(OSCAR_SEG_COST=$sc OSCAR_TAIL_COST=$tc timeout 300 python bench.py --config c3 --batch 256 --steps 8 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1))') c3_b64 $(OSCAR_SEG_COST=$sc OSCAR_TAIL_COST=$tc timeout 300 python bench.py --config c3 --batch 64 --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1))') C2 $(OSCAR_SEG_COST=$sc OSCAR_TAIL_COST=$tc timeout 200 python bench.py --steps 128 --warmup 8 --no-compare --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["us_per_step"],2))')"
done; done > $OUT/ab.txt 2>&1
