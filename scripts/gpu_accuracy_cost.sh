#!/bin/bash
# speed side of the accuracy/speed table: C2 attend (graph-replayed) per cost build, 3 rounds
mkdir -p gpurun_out/acc
bash scripts/variants.sh run base costb costk bytes2k > gpurun_out/acc/cost.txt 2>&1
