#!/bin/bash
mkdir -p gpurun_out/r2k
timeout 1200 python -m pytest tests/test_gpu_small.py tests/test_gpu_u8.py tests/test_gpu_edges.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/r2k/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2k/gputest.log
B="--no-cpu-baseline --steps 100"
for i in 1 2; do
for cfg in image_u8 image tiny; do
  timeout 300 python bench.py --config $cfg $B > gpurun_out/r2k/${cfg}_$i.json 2>&1
done
timeout 300 python bench.py --config image_u8 --mode avg $B > gpurun_out/r2k/image_u8avg_$i.json 2>&1
done
tail -3 gpurun_out/r2k/gputest.log
