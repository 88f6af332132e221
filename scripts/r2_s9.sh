#!/bin/bash
# column-major fused cls100: scanner rows staged (4 parts of 7 words) vs per-row stores
timeout 900 python -m pytest tests/test_gpu_colmajor.py tests/test_gpu_edges.py tests/test_gpu_shapes.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
LINES=("--config cls100 --layout col --steps 100" "--config cls100 --layout col --mode avg --steps 100" "--config cls100 --op scan --steps 100")
for v in "" cs0 ""; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
done
