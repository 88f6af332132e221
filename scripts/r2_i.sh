#!/bin/bash
mkdir -p gpurun_out/r2i
NCU_OUT=gpurun_out/r2i bash scripts/ncu_capture.sh image_u8_exact k_amm_rt --config image_u8 -- scale_exact k_amm_ws --config scale > gpurun_out/r2i/cap.log 2>&1
for t in image_u8_exact scale_exact; do
  ncu -i gpurun_out/r2i/prof_$t.ncu-rep --page details --csv > gpurun_out/r2i/details_$t.csv 2>&1
  ncu -i gpurun_out/r2i/prof_$t.ncu-rep --page raw --csv > gpurun_out/r2i/raw_$t.csv 2>&1
done
rm -f gpurun_out/r2i/*.ncu-rep.bak
