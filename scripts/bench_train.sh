#!/bin/bash
mkdir -p gpurun_out
for cfg in ${CONFIGS:-tiny cls10_c16 cls100 scale image}; do
  timeout 900 python bench.py --op train --config $cfg --steps 3 --warmup 1 --cpu-seconds 8 > gpurun_out/benchtrain_${cfg}.log 2>&1
  python - "$cfg" "gpurun_out/benchtrain_${cfg}.log" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], "gpu %.3e rows/s (%.1f ms)" % (d["value"], d["ms_per_step"]),
          "oracle %.3e rows/s" % d["cpu_baseline"]["value"])
except Exception as e:
    print(sys.argv[1], "ERR", e, open(sys.argv[2]).read()[-500:])
PY
done
