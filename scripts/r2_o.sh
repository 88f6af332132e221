#!/bin/bash
mkdir -p gpurun_out/r2o
timeout 1200 python -m pytest tests/test_gpu_small.py tests/test_gpu_u8.py tests/test_gpu_edges.py tests/test_gpu_parity.py tests/test_gpu_shapes.py -q -p no:cacheprovider -x > gpurun_out/r2o/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2o/gputest.log
B="--no-cpu-baseline --steps 100"
for i in 1 2; do
for v in main ll0; do
  L=libmaddness.so; [ $v != main ] && L=libmaddness_$v.so
  MDN_LIB=$L timeout 300 python bench.py --config image_u8 $B > gpurun_out/r2o/u8_${v}_$i.json 2>&1
  MDN_LIB=$L timeout 300 python bench.py --config image_u8 --mode avg $B > gpurun_out/r2o/u8avg_${v}_$i.json 2>&1
  MDN_LIB=$L timeout 300 python bench.py --config image $B > gpurun_out/r2o/image_${v}_$i.json 2>&1
  MDN_LIB=$L timeout 300 python bench.py --config tiny $B > gpurun_out/r2o/tiny_${v}_$i.json 2>&1
done
done
tail -3 gpurun_out/r2o/gputest.log
