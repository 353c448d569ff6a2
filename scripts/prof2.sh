for ctx in 1024 32768; do SWEEP_CTX=$ctx OSCAR_PROF=1 timeout 120 python scripts/sweep.py 2 2>&1 | grep -E "OSCAR_PROF|bits" | tail -3; done
