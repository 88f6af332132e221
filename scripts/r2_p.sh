#!/bin/bash
mkdir -p gpurun_out/r2p
B="--no-cpu-baseline --parity-rows 512 --steps 100"
for i in 1 2; do
for v in main nb2 nb4; do
  L=libmaddness.so; [ $v != main ] && L=libmaddness_$v.so
  for cfg in scale cls100 cls10_c32; do
    MDN_LIB=$L timeout 300 python bench.py --config $cfg $B > gpurun_out/r2p/${cfg}_${v}_$i.json 2>&1
  done
done
done
