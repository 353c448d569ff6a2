#!/bin/bash
# end-of-round headline refresh: smoke, the C2 line (value, e2e, roofline, cpu_baseline, comparisons), C1 line
export PYTHONUNBUFFERED=1
OUT=gpurun_out/fin; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --config c1 --steps 64 --warmup 4 > $OUT/bench_c1.json 2>/dev/null
