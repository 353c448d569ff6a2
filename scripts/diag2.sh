#!/bin/bash
mkdir -p gpurun_out
timeout 200 python scripts/diag_resid.py 2 2>&1 | tail -2 | tee gpurun_out/diag_resid2.txt
timeout 200 python scripts/diag_resid.py 4 2>&1 | tail -2 | tee -a gpurun_out/diag_resid2.txt
OSCAR_PROF=1 timeout 120 python scripts/sweep.py 2 2>&1 | grep -E "OSCAR_PROF|bits" | tail -3 | tee gpurun_out/diag_prof.txt
