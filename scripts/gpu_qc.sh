#!/bin/bash
# quantize: the quad chain's step loop rolled (smaller code, OSK_QC_ROLL=1 variant) vs unrolled; C3 B=8 line refresh
export PYTHONUNBUFFERED=1
OUT=gpurun_out/qc; mkdir -p $OUT
Q=$PWD/paper_2605_19660_b200/liboscar_b200_qc.so; N=$PWD/paper_2605_19660_b200/liboscar_b200.so
for r in 1 2; do for v in base qc; do L=$N; [ $v = qc ] && L=$Q
  echo "$v $(OSCAR_LIB=$L timeout 300 python scripts/diag_prefill.py 2>/dev/null | tail -1)"
done; done > $OUT/ab.txt 2>&1
timeout 900 python bench.py --config c3 --batch 8 --steps 16 --warmup 3 > $OUT/bench_c3_b8.json 2>/dev/null
