#!/bin/bash
# Column-major encode-only: TMA-gather4 warp-specialised kernel vs thread-per-row kernel.
mkdir -p gpurun_out
for cfg in cls100 scale cls10_c16; do
  for ws in 1 0; do
    MDN_CM_WS_ENCODE=$ws timeout 300 python bench.py --layout col --op encode --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cme.log 2>&1
    python -c "
import json;d=json.loads(open('gpurun_out/cme.log').read().strip().splitlines()[-1]);print('$cfg encode ws=$ws', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'])" 2>&1 | tail -1
  done
done
