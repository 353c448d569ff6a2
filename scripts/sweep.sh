mkdir -p gpurun_out
for bits in 2 4 0; do for ncw in 8 12; do for pf in 0 8; do
  OSCAR_NCW=$ncw OSCAR_L2_PREFETCH=$pf timeout 120 python scripts/sweep.py $bits 2>&1 | tail -1
done; done; done | tee gpurun_out/sweep.txt
