#!/bin/bash
# Column-major (N2) A/B: warp-specialised TMA-gather4 kernel (default) vs the thread-per-row kernel.
mkdir -p gpurun_out
for cfg in ${CONFIGS:-tiny image cls10_c16 scale cls100}; do
  for simple in 0 1; do
    MDN_CM_SIMPLE=$simple timeout 300 python bench.py --layout col --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cmr.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/cmr.log').read().strip().splitlines()[-1]);print('$cfg simple=$simple', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'])" 2>&1 | tail -1
  done
done
