#!/bin/bash
mkdir -p gpurun_out/r2m
python bench.py --config image_u8 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2m/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_amm_rt -s 1 -c 1 -f -o /tmp/prof_u8 python bench.py --config image_u8 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2m/ncu.log 2>&1
ncu -i /tmp/prof_u8.ncu-rep --page source --csv --print-source sass > gpurun_out/r2m/src.csv 2>&1
ncu -i /tmp/prof_u8.ncu-rep --page raw --csv > gpurun_out/r2m/raw.csv 2>&1
python scripts/ncu_summary.py full /tmp/prof_u8.ncu-rep gpurun_out/r2m/ncu_full_image_u8_exact.json > /dev/null 2>&1
