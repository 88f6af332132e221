#!/bin/bash
# ncu --set full of one k_amm launch for a bench config (after a plain run of the same command).
# usage: CFG=image_u8 MODE=exact KERNEL=k_amm bash scripts/ncu_one.sh
set -e
mkdir -p gpurun_out
CMD="python bench.py --config ${CFG} --mode ${MODE:-exact} --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/plain_${CFG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_amm} -s 1 -c 1 \
    -o gpurun_out/prof_${CFG}_${MODE:-exact}${TAG} $CMD > gpurun_out/ncu_${CFG}.log 2>&1
