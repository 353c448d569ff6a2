#!/bin/bash
# TILES kernel at many-segment launches (> 2 segments per CTA, where DEFER runs): OSCAR_TILE_UNITS=3 vs default
export PYTHONUNBUFFERED=1
OUT=gpurun_out/tiles7; mkdir -p $OUT
OSCAR_TILE_UNITS=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_shapes.py tests/test_gpu_scale.py -q -x > $OUT/pytest_tu3.txt 2>&1; echo "rc=$?" >> $OUT/pytest_tu3.txt
for r in 1 2; do for tu in 1 3; do
  echo "tu$tu c3_b256 $(OSCAR_TILE_UNITS=$tu timeout 300 python bench.py --config c3 --batch 256 --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1), round(d["roofline"]["frac"],3))')"
  echo "tu$tu c3_proxy2 $(OSCAR_TILE_UNITS=$tu timeout 300 python bench.py --config c3 --proxy-world 2 --steps 16 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"]*1e3,1))')"
done; done > $OUT/ab.txt 2>&1
