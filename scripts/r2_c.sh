#!/bin/bash
mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_probe.py -q -p no:cacheprovider > gpurun_out/r2c/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c/gputest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2c/default.json 2> gpurun_out/r2c/default.err
for cfg in cls100 scale cls10_c16 cls10_c64; do
 for mode in exact avg; do
  timeout 600 python bench.py --config $cfg --mode $mode --no-cpu-baseline > gpurun_out/r2c/${cfg}_$mode.json 2> gpurun_out/r2c/${cfg}_$mode.err
 done
done
tail -3 gpurun_out/r2c/gputest.log
