#!/bin/bash
# Multi-GPU configs on one B200: per-rank shard proxies of 2/4/8-GPU runs
# (bench.py --proxy-world N), the whole configs on one GPU, the C3 batch sweep
#   gpurun -- 'bash scripts/gpu_proxies.sh'   -> gpurun_out/proxy/
export PYTHONUNBUFFERED=1
OUT=gpurun_out/proxy; mkdir -p $OUT
for n in 8 4 2; do
  timeout 600 python bench.py --config c3 --proxy-world $n --steps 16 --warmup 3 > $OUT/c3_$n.json 2> $OUT/c3_$n.err
  timeout 600 python bench.py --config c4 --proxy-world $n --steps 32 --warmup 4 > $OUT/c4_$n.json 2> $OUT/c4_$n.err
  timeout 600 python bench.py --config c5 --proxy-world $n --steps 32 --warmup 4 > $OUT/c5_$n.json 2> $OUT/c5_$n.err
done
for c in c4 c5; do timeout 600 python bench.py --config $c --steps 64 --warmup 4 > $OUT/${c}_1.json 2> $OUT/${c}_1.err; done
for b in 256 64 8 1; do timeout 900 python bench.py --config c3 --batch $b --steps 16 --warmup 3 > $OUT/c3_b$b.json 2>/dev/null; done
