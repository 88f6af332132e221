#!/bin/bash
# Column-major (N2) A/B: rows per stage R of the warp-specialised variant vs the thread-per-row kernel.
mkdir -p gpurun_out
one() {  # label, env..., -- bench args
  local label=$1; shift
  env "$@" timeout 300 python bench.py --layout col --steps 10 --warmup 3 --no-cpu-baseline $BARGS > gpurun_out/cmr.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/cmr.log').read().strip().splitlines()[-1]);print('$label', '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'])" 2>&1 | tail -1
}
for cfg in cls100 scale cls10_c16; do
  BARGS="--config $cfg"
  for R in 64 128 256; do one "$cfg ws R=$R" MDN_CM_WS=1 MDN_CM_R=$R; done
  one "$cfg simple" MDN_CM_SIMPLE=1
done
