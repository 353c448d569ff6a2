#!/bin/bash
# One GPU round: parity tests, smoke, bench, ncu launch list + one full capture.
set -x
mkdir -p gpurun_out; rm -f gpurun_out/parity_errors.jsonl
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -30 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_attn|quantize_kernel|raw_block|ring_copy|lse_merge" -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 16 --warmup 2 --no-compare --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_attn -s 3 -c 1 \
  -o gpurun_out/prof_attn_int2 -f python bench.py --steps 8 --warmup 2 --no-compare --no-cpu > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quantize_kernel -c 1 \
  -o gpurun_out/prof_quant_int2 -f python bench.py --steps 2 --warmup 1 --no-compare --no-cpu > gpurun_out/ncu_quant.log 2>&1
fi
ls -la gpurun_out
