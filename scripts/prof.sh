for cfg in "2 12" "2 8" "4 8"; do set -- $cfg
  OSCAR_PROF=1 OSCAR_NCW=$2 timeout 120 python scripts/sweep.py $1 2>&1 | grep -E "OSCAR_PROF|bits" | tail -3
done
for ctx in 16384 65536; do SWEEP_CTX=$ctx timeout 120 python scripts/sweep.py 2 | tail -1; done
