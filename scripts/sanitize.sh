#!/bin/bash
mkdir -p gpurun_out/san
python scripts/sanitize_all.py > gpurun_out/san/plain.txt 2>&1; tail -4 gpurun_out/san/plain.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_all.py > gpurun_out/san/$tool.txt 2>&1
  echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok " gpurun_out/san/$tool.txt | tail -6
done
