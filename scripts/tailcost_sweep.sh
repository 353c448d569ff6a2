#!/bin/bash
# attend latency vs residual fill r for several OSCAR_TAIL_COST values (C2 INT2)
for tc in ${TCS:-0 3 6 10 16}; do
  echo "tail_cost=$tc $(OSCAR_TAIL_COST=$tc timeout 200 python scripts/diag_resid.py 2 | tail -1)"
done
