#!/bin/bash
mkdir -p gpurun_out/r2d
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_probe.py tests/test_gpu_edges.py -q -p no:cacheprovider -x > gpurun_out/r2d/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d/gputest.log
B="--no-cpu-baseline --parity-rows 0 --steps 50"
for cfg in scale cls10_c16 cls10_c32; do
  timeout 300 python bench.py --config $cfg $B > gpurun_out/r2d/${cfg}_def.json 2>&1
  MDN_SUBF_SLABS=0 timeout 300 python bench.py --config $cfg $B > gpurun_out/r2d/${cfg}_noslab.json 2>&1
  MDN_LIB=libmaddness_s8.so timeout 300 python bench.py --config $cfg $B > gpurun_out/r2d/${cfg}_s8.json 2>&1
  MDN_LIB=libmaddness_e8s8.so timeout 300 python bench.py --config $cfg $B > gpurun_out/r2d/${cfg}_e8s8.json 2>&1
done
timeout 300 python bench.py --config scale --op encode $B > gpurun_out/r2d/scale_enc_def.json 2>&1
MDN_SUBF_SLABS=0 timeout 300 python bench.py --config scale --op encode $B > gpurun_out/r2d/scale_enc_noslab.json 2>&1
tail -3 gpurun_out/r2d/gputest.log
