#!/bin/bash
# same-box A/B of decode steps (C2 hot/cold inputs, C3 small batch)
for r in 1 2; do for lib in old new; do L=$PWD/paper_2605_19660_b200/liboscar_b200_$lib.so
  echo "$lib C2decode $(OSCAR_LIB=$L timeout 200 python scripts/diag_hot.py | tail -1)"
  for b in ${AB_C3B:-1 8}; do echo "$lib C3b$b $(OSCAR_LIB=$L timeout 200 python scripts/diag_c3.py $b | tail -1)"; done
done; done
