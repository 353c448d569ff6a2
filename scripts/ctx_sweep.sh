for ctx in 1024 4096 8192 16384 32768 65536; do SWEEP_CTX=$ctx timeout 120 python scripts/sweep.py 2 | tail -1; done
for ctx in 1024 32768; do SWEEP_CTX=$ctx timeout 120 python scripts/sweep.py 0 | tail -1; done
