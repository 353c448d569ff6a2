#!/bin/bash
# C2 headline bench (full) + the C3/C4/C5 config lines at N=1
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -3 gpurun_out/bench_c2.err
for c in c4 c5; do timeout 600 python bench.py --config $c --steps 64 --warmup 4 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
for b in 256 64 8 1; do timeout 900 python bench.py --config c3 --batch $b --steps 16 --warmup 3 > gpurun_out/bench_c3_b$b.json 2> gpurun_out/bench_c3_b$b.err; tail -2 gpurun_out/bench_c3_b$b.err; done
for f in gpurun_out/bench_c*.json; do echo $f; python -c "
import json,sys
d=json.load(open('$f'))
print(round(d['value'],1), d['unit'], 'ms/step', round(d['ms_per_step'],4), 'frac', round(d['roofline']['frac'],3), d['config'].get('workload','')[:60])
"; done
