#!/bin/bash
mkdir -p gpurun_out/r2b
timeout 1200 python -m pytest tests/test_gpu_bench.py tests/test_gpu_edges.py tests/test_gpu_pq.py -q -p no:cacheprovider --timeout 900 > gpurun_out/r2b/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2b/gputest.log
timeout 600 python bench.py > gpurun_out/r2b/default.json 2> gpurun_out/r2b/default.err
for cfg in cls100 scale tiny cls10_c16; do
  timeout 600 python bench.py --config $cfg --op encode --encoder pq --no-cpu-baseline > gpurun_out/r2b/pq_$cfg.json 2> gpurun_out/r2b/pq_$cfg.err
done
timeout 300 python bench.py --gpus 2 --steps 20 > gpurun_out/r2b/gpus2_nccl.json 2> gpurun_out/r2b/gpus2_nccl.err; echo "nccl2 rc=$?" >> gpurun_out/r2b/gpus2_nccl.err
tail -3 gpurun_out/r2b/gputest.log
