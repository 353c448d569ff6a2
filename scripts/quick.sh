mkdir -p gpurun_out; rm -f gpurun_out/parity_errors.jsonl
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 2>&1 | tail -4
for cfg in "2 12" "2 8" "4 8" "4 12" "0 12"; do set -- $cfg
  OSCAR_NCW=$2 timeout 120 python scripts/sweep.py $1 2>&1 | tail -1
done
