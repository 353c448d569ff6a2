#!/bin/bash
# parity tests + attention timing vs residual fill + flush timing + bench
mkdir -p gpurun_out; rm -f gpurun_out/parity_errors.jsonl
export PYTHONUNBUFFERED=1
if [ "${TESTS:-1}" = "1" ]; then
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -15 gpurun_out/pytest_gpu.txt
fi
for b in ${BITS:-2}; do timeout 200 python scripts/diag_resid.py $b 2>&1 | tail -1; done | tee gpurun_out/diag_resid.txt
timeout 200 python scripts/diag_flush.py 2>&1 | tail -1 | tee gpurun_out/diag_flush.txt
timeout 600 python bench.py --no-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; tail -2 gpurun_out/bench_quick.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_quick.json'))
print({k: d[k] for k in ('value','us_per_step','host_us_per_step','flush_step_us')}, d['roofline']['avg_launch_us'], d['roofline']['frac'], d['e2e']['us_per_step'], d['clocks']['sm_mhz'], {k:(v.get('attn_kernel_us') if isinstance(v,dict) else v) for k,v in d.get('comparisons',{}).items()})
PY
