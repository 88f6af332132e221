#!/bin/bash
# Bench every config in both modes (1 GPU); one JSON line per run in gpurun_out/.
mkdir -p gpurun_out
for cfg in ${CONFIGS:-cls100 cls10_c16 cls10_c32 cls10_c64 scale tiny image}; do
  for mode in exact avg; do
    timeout 600 python bench.py --config $cfg --mode $mode --steps 20 --warmup 3 --no-cpu-baseline \
      > gpurun_out/bench_${cfg}_${mode}.log 2>&1 || echo "FAILED $cfg $mode" >> gpurun_out/bench_all_fail.txt
  done
done
