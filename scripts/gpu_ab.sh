#!/bin/bash
# Same-box A/B of the working tree against HEAD plus the GPU tests and the
# profiling-build timelines.  Build first (here): scripts/abbuild.sh (writes
# liboscar_b200_old.so from HEAD, liboscar_b200_new.so from the working tree)
# and `make -C paper_2605_19660_b200/csrc PROF=1`.
#   gpurun -- 'bash scripts/gpu_ab.sh'   -> gpurun_out/ab/
export PYTHONUNBUFFERED=1
OUT=gpurun_out/ab; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for r in 1 2; do for v in old new; do L=$PWD/paper_2605_19660_b200/liboscar_b200_$v.so
  echo "$v C2 $(OSCAR_LIB=$L timeout 200 python scripts/sweep.py 2 | tail -1)"
  for b in 1 8; do echo "$v C3b$b $(OSCAR_LIB=$L timeout 200 python scripts/diag_c3.py $b | tail -1)"; done
  echo "$v C5p8 $(OSCAR_LIB=$L timeout 200 python scripts/diag_c5proxy.py 8 | tail -1)"
done; done > $OUT/ab.txt 2>&1
timeout 300 python bench.py --steps 64 --warmup 8 --no-compare --no-cpu > $OUT/bench_c2.json 2>&1
export OSCAR_PROF=1 OSCAR_LIB=$PWD/paper_2605_19660_b200/liboscar_b200_prof.so
for spec in "8192 1 2 28 4" "8192 8 2 28 4" "131072 8 2 4 1" "32768 16 2 32 8"; do
  echo "=== $spec" ; timeout 300 python scripts/diag_timeline.py $spec 2>&1 | grep -v "^---" | tail -5
done > $OUT/timelines.txt 2>&1
