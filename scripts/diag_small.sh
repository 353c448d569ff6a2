for cfg in "1 8192" "8 8192" "64 8192" "1 524288"; do timeout 120 python scripts/diag_small.py $cfg 2>&1 | tail -1; done
for cfg in "1 8192" "1 524288"; do OSCAR_PROF=1 timeout 120 python scripts/diag_small.py $cfg 2>&1 | grep OSCAR_PROF | tail -2; done
