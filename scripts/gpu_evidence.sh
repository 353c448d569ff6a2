#!/bin/bash
# Round evidence in one GPU call: parity tests, smoke, the headline bench,
# config lines, ncu launch list of the bench + full captures of the two kernels.
set -x
OUT=gpurun_out/ev; mkdir -p $OUT; rm -f gpurun_out/parity_errors.jsonl
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > $OUT/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.txt
cp gpurun_out/parity_errors.jsonl $OUT/ 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in c1 c4 c5; do timeout 600 python bench.py --config $c --steps 64 --warmup 4 > $OUT/bench_$c.json 2>/dev/null; done
for b in 256 64 8 1; do timeout 900 python bench.py --config c3 --batch $b --steps 16 --warmup 3 > $OUT/bench_c3_b$b.json 2>/dev/null; done
for b in 4 0; do timeout 200 python scripts/diag_resid.py $b 2>/dev/null | tail -1; done > $OUT/attend_by_residual.txt
timeout 200 python scripts/diag_resid.py 2 2>/dev/null | tail -1 >> $OUT/attend_by_residual.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"decode_attn|quantize_kernel|raw_block|ring_copy|lse_merge" -c 80 --csv --log-file $OUT/launches_bench.csv \
  python bench.py --steps 32 --warmup 3 --no-compare --no-cpu > $OUT/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 12 -c 1 \
  -o $OUT/prof_attn_int2 -f python scripts/sweep.py 2 > $OUT/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 12 -c 1 \
  -o $OUT/prof_attn_int4 -f python scripts/sweep.py 4 > $OUT/ncu_attn4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize_kernel -s 4 -c 1 \
  -o $OUT/prof_quant_int2 -f python bench.py --steps 2 --warmup 1 --no-compare --no-cpu > $OUT/ncu_quant.log 2>&1
ls -la $OUT
