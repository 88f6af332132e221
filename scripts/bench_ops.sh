#!/bin/bash
# Unfused halves (mdn_encode, mdn_scan) per config, exact mode.
mkdir -p gpurun_out
for cfg in ${CONFIGS:-cls100 cls10_c16 scale tiny image}; do
  for op in encode scan; do
    timeout 600 python bench.py --config $cfg --op $op --steps 20 --warmup 3 --no-cpu-baseline \
      > gpurun_out/ops_${cfg}_${op}.log 2>&1
  done
done
