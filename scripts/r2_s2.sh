#!/bin/bash
# wide-table mdn_scan: threads per one-per-SM block (256 / 384 / 512) at the same register budget
for v in "" t384 t512 ""; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "--config cls100 --op scan --steps 100" "--config cls100 --op scan --mode avg --steps 100" "--config cls10_c64 --op scan --steps 100" "--config cls100 --layout col --steps 100" 2>&1 | cut -c1-150
done
MDN_LIB=libmaddness_t512.so timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
