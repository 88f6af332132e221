#!/bin/bash
# raw-word exact scan (MDN_SCAN_RAW=1) vs the mask form (raw0): full GPU suite, scan / col / fused lines
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_raw.log 2>&1; tail -1 gpurun_out/pytest_raw.log
LINES=("--config cls100 --op scan --steps 100" "--config cls10_c64 --op scan --steps 100" "--config cls10_c32 --op scan --steps 100" "--config scale --op scan --steps 100" "--config cls10_c16 --op scan --steps 100" "--config cls100 --layout col --steps 100" "--config scale --layout col --steps 100" "--config cls100 --steps 100" "--config scale --steps 100" "--config cls10_c16 --layout col --steps 100")
for v in "" raw0; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
done
