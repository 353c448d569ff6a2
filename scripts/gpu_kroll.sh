#!/bin/bash
# quantize: K-side group loops unrolled 4 / 8 (OSK_KROLL variants) vs 32; GPU tests of the default build
export PYTHONUNBUFFERED=1
OUT=gpurun_out/kroll; mkdir -p $OUT
N=$PWD/paper_2605_19660_b200/liboscar_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for r in 1 2; do for v in base kr4 kr8; do L=$N; [ $v != base ] && L=$PWD/paper_2605_19660_b200/liboscar_b200_$v.so
  echo "$v $(OSCAR_LIB=$L timeout 300 python scripts/diag_prefill.py 2>/dev/null | tail -1)"
done; done > $OUT/ab.txt 2>&1
