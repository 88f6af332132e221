#!/bin/bash
mkdir -p gpurun_out/r2n
timeout 1200 python -m pytest tests/test_gpu_pq.py -q -p no:cacheprovider -x > gpurun_out/r2n/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2n/gputest.log
B="--no-cpu-baseline --steps 30 --op encode --encoder pq"
for v in main pqf0; do
  L=libmaddness.so; [ $v != main ] && L=libmaddness_$v.so
  for cfg in cls100 scale tiny cls10_c16; do
    MDN_LIB=$L timeout 300 python bench.py --config $cfg $B > gpurun_out/r2n/${cfg}_$v.json 2>&1
  done
done
tail -3 gpurun_out/r2n/gputest.log
