#!/bin/bash
# TILES kernel forced for every launch (OSCAR_TILE_UNITS=2) vs the default selection, per config
mkdir -p gpurun_out/tiles5
for tu in 1 2; do
  for c in c4 c5; do echo "tu$tu ${c}_1gpu $(OSCAR_TILE_UNITS=$tu timeout 300 python bench.py --config $c --steps 64 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"; done
  for c in c4 c3; do echo "tu$tu ${c}_proxy4 $(OSCAR_TILE_UNITS=$tu timeout 300 python bench.py --config $c --proxy-world 4 --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"; done
  echo "tu$tu c4_proxy8 $(OSCAR_TILE_UNITS=$tu timeout 300 python bench.py --config c4 --proxy-world 8 --steps 32 --warmup 4 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,2))')"
done > gpurun_out/tiles5/ab.txt 2>&1
