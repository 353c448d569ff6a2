#!/bin/bash
# same-box A/B of the C5 step (bench.py --config c5) between liboscar_b200_{old,new}.so
for r in 1 2; do for lib in old new; do L=$PWD/paper_2605_19660_b200/liboscar_b200_$lib.so
  echo "$lib C5 $(OSCAR_LIB=$L timeout 300 python bench.py --config c5 --steps 64 --warmup 4 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,2), "us", round(d["roofline"]["frac"],3))')"
done; done
