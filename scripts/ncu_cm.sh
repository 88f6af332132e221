#!/bin/bash
set -e
mkdir -p gpurun_out
CMD="python bench.py --layout col --config cls100 --steps 2 --warmup 1 --no-cpu-baseline"
MDN_CM_R=128 $CMD > gpurun_out/plain_cm.log 2>&1
MDN_CM_R=128 ncu --set full --clock-control none --import-source on -k regex:k_amm -s 1 -c 1 -o gpurun_out/prof_cm_cls100 $CMD > gpurun_out/ncu_cm.log 2>&1
