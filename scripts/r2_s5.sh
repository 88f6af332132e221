#!/bin/bash
# 8-byte table loads in the exact scan (MDN_SCAN_PAIR 1 = W >= 8, 2 = W >= 2, 0 = off)
timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py tests/test_gpu_tiled.py -m gpu -q -x 2>&1 | tail -1
MDN_LIB=libmaddness_p2.so timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
LINES=("--config cls100 --op scan --steps 100" "--config cls100 --op scan --mode avg --steps 100" "--config cls10_c64 --op scan --steps 100" "--config cls10_c32 --op scan --steps 100" "--config scale --op scan --steps 100" "--config cls10_c16 --op scan --steps 100")
for v in "" p0 p2; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
done
export NCU_OUT=/tmp NCU_SUMMARY=1
bash scripts/ncu_capture.sh scan_pair k_scan_fast --config cls100 --op scan
