#!/bin/bash
# PQ comparator vs MADDNESS encode, same configs.
mkdir -p gpurun_out
for cfg in ${CONFIGS:-cls100 cls10_c16 scale tiny}; do
  for enc in maddness pq; do
    timeout 300 python bench.py --op encode --encoder $enc --config $cfg --steps 10 --warmup 3 --no-cpu-baseline \
      > gpurun_out/benchenc_${enc}_${cfg}.log 2>&1
    python - "$cfg" "$enc" "gpurun_out/benchenc_${enc}_${cfg}.log" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[1], sys.argv[2], "encode %.3e rows/s" % d["value"], "%s frac=%.3f" % (r["bound"], r["frac"]))
except Exception as e:
    print(sys.argv[1], sys.argv[2], "ERR", e)
PY
  done
done
timeout 300 python bench.py --encoder pq --config cls100 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/benchpq_amm_cls100.log 2>&1
tail -1 gpurun_out/benchpq_amm_cls100.log | cut -c1-300
