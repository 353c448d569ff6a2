#!/bin/bash
# same-box A/B of two builds: liboscar_b200_old.so vs liboscar_b200_new.so
for r in 1 2; do for lib in old new; do L=$PWD/paper_2605_19660_b200/liboscar_b200_$lib.so
  echo "$lib C2attend $(OSCAR_LIB=$L timeout 100 python scripts/sweep.py 2 | tail -1 | python -c 'import json,sys; print(json.load(sys.stdin)["us"])')"
  for b in ${AB_C3B:-1 8}; do echo "$lib C3b$b $(OSCAR_LIB=$L timeout 200 python scripts/diag_c3.py $b | tail -1)"; done
  [ -n "$AB_RESID" ] && echo "$lib resid $(OSCAR_LIB=$L timeout 200 python scripts/diag_resid.py 2 | tail -1)"
done; done
