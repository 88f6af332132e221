#!/bin/bash
mkdir -p gpurun_out/r2e
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -q -p no:cacheprovider -x -k "scan or Scan or shapes" > gpurun_out/r2e/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2e/gputest.log
B="--no-cpu-baseline --parity-rows 0 --steps 50 --op scan"
for cfg in cls100 scale cls10_c16 cls10_c64 tiny image; do
  timeout 300 python bench.py --config $cfg $B > gpurun_out/r2e/${cfg}_pf1.json 2>&1
  MDN_LIB=libmaddness_pf0.so timeout 300 python bench.py --config $cfg $B > gpurun_out/r2e/${cfg}_pf0.json 2>&1
done
timeout 300 python bench.py --config cls100 $B --mode avg > gpurun_out/r2e/cls100avg_pf1.json 2>&1
MDN_LIB=libmaddness_pf0.so timeout 300 python bench.py --config cls100 $B --mode avg > gpurun_out/r2e/cls100avg_pf0.json 2>&1
tail -3 gpurun_out/r2e/gputest.log
