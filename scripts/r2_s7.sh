#!/bin/bash
# mdn_scan wide tables: output rows staged through shared memory (coalesced stores) vs per-row float4 stores
timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py tests/test_gpu_tiled.py tests/test_gpu_small.py -m gpu -q -x 2>&1 | tail -1
LINES=("--config cls100 --op scan --steps 100" "--config cls100 --op scan --mode avg --steps 100")
for v in "" st0 ""; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
done
export NCU_OUT=/tmp NCU_SUMMARY=1
bash scripts/ncu_capture.sh scan_staged k_scan_fast --config cls100 --op scan
