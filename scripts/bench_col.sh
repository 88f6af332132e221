#!/bin/bash
# Column-major A bench lines, both modes.
mkdir -p gpurun_out
for cfg in ${CONFIGS:-cls100 scale cls10_c16 tiny}; do
  for mode in exact avg; do
    timeout 300 python bench.py --layout col --config $cfg --mode $mode --steps 20 --warmup 3 --no-cpu-baseline \
      > gpurun_out/benchcol_${cfg}_${mode}.log 2>&1 || echo "FAILED $cfg $mode" >> gpurun_out/bench_fail.txt
    python - "$cfg" "$mode" "gpurun_out/benchcol_${cfg}_${mode}.log" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], "%.3e" % d["value"], "frac=%.3f" % d["roofline"]["frac"],
          "B/row=%d" % (d["roofline"]["algorithmic_bytes_per_launch"] // d["config"]["rows_per_gpu"]))
except Exception as e:
    print(sys.argv[1], sys.argv[2], "ERR", e)
PY
  done
done
