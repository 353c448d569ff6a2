mkdir -p gpurun_out/e2e
for r in 1 2; do for m in 0 1; do
  echo "mode$m $(OSCAR_HOST_INPUTS=$m timeout 300 python bench.py --steps 64 --warmup 8 --no-compare --no-cpu 2>/dev/null | python -c 'import json,sys; d=json.load(sys.stdin); print(d["us_per_step"], d["e2e"]["us_per_step"])')"
done; done > gpurun_out/e2e/ab.txt 2>&1
OSCAR_HOST_INPUTS=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -k host > gpurun_out/e2e/pytest.txt 2>&1
