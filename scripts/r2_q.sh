#!/bin/bash
mkdir -p gpurun_out/r2q
B="--no-cpu-baseline --parity-rows 4096 --steps 100"
for i in 1 2; do
for v in main cta2; do
  L=libmaddness.so; [ $v != main ] && L=libmaddness_$v.so
  MDN_LIB=$L timeout 300 python bench.py --config image_u8 $B > gpurun_out/r2q/u8_${v}_$i.json 2>&1
  MDN_LIB=$L timeout 300 python bench.py --config image_u8 --op encode $B > gpurun_out/r2q/u8enc_${v}_$i.json 2>&1
  MDN_LIB=$L timeout 300 python bench.py --config image_u8 --mode avg $B > gpurun_out/r2q/u8avg_${v}_$i.json 2>&1
done
done
