#!/bin/bash
# mdn_scan wide tables: TMA tensor stores of the staged rows (MDN_SCAN_TSTORE, 1 or 2 buffers per warp) vs LDS + STG readback
for v in ts1 ts2; do
  echo "== tests $v"
  MDN_LIB=libmaddness_$v.so timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py tests/test_gpu_tiled.py tests/test_gpu_edges.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
done
LINES=("--config cls100 --op scan --steps 100" "--config cls100 --op scan --mode avg --steps 100")
for v in "" ts1 ts2 "" ts1; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
done
export NCU_OUT=/tmp NCU_SUMMARY=1
MDN_LIB=libmaddness_ts1.so bash scripts/ncu_capture.sh scan_ts1 k_scan_ts --config cls100 --op scan
MDN_LIB=libmaddness_ts2.so bash scripts/ncu_capture.sh scan_ts2 k_scan_ts --config cls100 --op scan
ls gpurun_out/
