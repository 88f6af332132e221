#!/bin/bash
mkdir -p gpurun_out/r2h
B="--no-cpu-baseline --parity-rows 4096 --steps 30 --op encode --encoder pq"
for v in main pqa pqb pqc; do
  L=libmaddness.so; [ $v != main ] && L=libmaddness_$v.so
  for cfg in cls100 scale tiny cls10_c16; do
    MDN_LIB=$L timeout 300 python bench.py --config $cfg $B > gpurun_out/r2h/${cfg}_$v.json 2>&1
  done
done
