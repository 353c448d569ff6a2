#!/bin/bash
# one ncu --set full capture of the INT2 attention kernel (C2 attend, graph-free) + launch list of a bench run
mkdir -p gpurun_out
TAG=${TAG:-r01b}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 12 -c 1 \
  -o gpurun_out/prof_attn_$TAG -f python scripts/sweep.py 2 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"decode_attn|quantize_kernel|ring_copy|lse_merge" -c 60 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 32 --warmup 3 --no-compare --no-cpu > gpurun_out/ncu_bench_$TAG.log 2>&1
ls -la gpurun_out | grep $TAG
