#!/bin/bash
# Bench the small-row configs (tiny, image, image_u8) in both modes; one JSON line each.
mkdir -p gpurun_out
for cfg in ${CONFIGS:-tiny image image_u8}; do
  for mode in exact avg; do
    timeout 300 python bench.py --config $cfg --mode $mode --steps 20 --warmup 3 --no-cpu-baseline \
      > gpurun_out/bench_${cfg}_${mode}${TAG}.log 2>&1 || echo "FAILED $cfg $mode" >> gpurun_out/bench_fail.txt
    python - "$cfg" "$mode" "gpurun_out/bench_${cfg}_${mode}${TAG}.log" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], "%.3e" % d["value"], "frac=%.3f" % d["roofline"]["frac"], d["roofline"]["kernel"])
except Exception as e:
    print(sys.argv[1], sys.argv[2], "ERR", e)
PY
  done
done
