#!/bin/bash
# tests + timing diagnostics + bench + config lines (one GPU call)
bash scripts/gpu_quick.sh
for c in c4 c5; do timeout 600 python bench.py --config $c --steps 64 --warmup 4 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
for b in ${C3B:-256 1}; do timeout 900 python bench.py --config c3 --batch $b --steps 16 --warmup 3 > gpurun_out/bench_c3_b$b.json 2> gpurun_out/bench_c3_b$b.err; tail -2 gpurun_out/bench_c3_b$b.err; done
for f in gpurun_out/bench_c[345]*.json; do python -c "
import json,sys
d=json.load(open('$f'))
print('$f', round(d['value'],1), d['unit'], 'ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3))
"; done
