#!/bin/bash
mkdir -p gpurun_out/r2f
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -q -p no:cacheprovider -x > gpurun_out/r2f/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2f/gputest.log
B="--no-cpu-baseline --parity-rows 0 --steps 50 --op scan"
for cfg in cls100 scale cls10_c16 cls10_c32 cls10_c64; do
  timeout 300 python bench.py --config $cfg $B > gpurun_out/r2f/${cfg}_auto.json 2>&1
  MDN_LIB=libmaddness_pf1.so timeout 300 python bench.py --config $cfg $B > gpurun_out/r2f/${cfg}_pf1.json 2>&1
  MDN_LIB=libmaddness_pf0.so timeout 300 python bench.py --config $cfg $B > gpurun_out/r2f/${cfg}_pf0.json 2>&1
done
for m in auto pf1 pf0; do
  L=libmaddness.so; [ $m != auto ] && L=libmaddness_$m.so
  MDN_LIB=$L timeout 300 python bench.py --config cls100 $B --mode avg > gpurun_out/r2f/cls100avg_$m.json 2>&1
done
tail -3 gpurun_out/r2f/gputest.log
