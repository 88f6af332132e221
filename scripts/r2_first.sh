#!/bin/bash
# round 2, first box: full GPU suite, default bench, PQ lines, 2-rank self-launch
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r2a/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a/gputest.log
timeout 600 python bench.py > gpurun_out/r2a/default.json 2> gpurun_out/r2a/default.err
for cfg in cls100 scale tiny cls10_c16; do
  timeout 600 python bench.py --config $cfg --op encode --encoder pq --no-cpu-baseline > gpurun_out/r2a/pq_$cfg.json 2> gpurun_out/r2a/pq_$cfg.err
done
timeout 600 python bench.py --gpus 2 --steps 20 > gpurun_out/r2a/gpus2_nccl.json 2> gpurun_out/r2a/gpus2_nccl.err
tail -3 gpurun_out/r2a/gputest.log
