#!/bin/bash
# raw-form averaging split; column-major scanners ALU-only (cm0) vs mix 3
timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py tests/test_gpu_colmajor.py tests/test_gpu_tiled.py -m gpu -q -x 2>&1 | tail -1
LINES=("--config cls100 --op scan --mode avg --steps 100" "--config cls100 --mode avg --steps 100" "--config cls100 --layout col --steps 100" "--config cls100 --layout col --mode avg --steps 100" "--config scale --layout col --steps 100")
for v in "" cm0; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
done
