#!/bin/bash
# raw-word scan: pipe mix of the odd-lane adds (MIXK 2 / 3 / 5 / 64, 0 = ALU only) + ncu of the cls100 scan
LINES=("--config cls100 --op scan --steps 100" "--config cls10_c64 --op scan --steps 100" "--config scale --op scan --steps 100" "--config cls100 --layout col --steps 100")
for v in "" m2 m5 m64; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
done
echo "== MIX 0 (ALU only)"
MDN_SCAN_MIX=0 python scripts/bench_lines.py "${LINES[@]:0:3}" "--config cls10_c16 --op scan --steps 100" 2>&1 | cut -c1-150
echo "== MIX 3 forced (C = 16 too)"
MDN_SCAN_MIX=3 python scripts/bench_lines.py "--config cls10_c16 --op scan --steps 100" "--config image --op scan --steps 100" "--config tiny --op scan --steps 100" 2>&1 | cut -c1-150
python scripts/bench_lines.py "--config cls10_c16 --op scan --steps 100" "--config image --op scan --steps 100" "--config tiny --op scan --steps 100" 2>&1 | cut -c1-150
export NCU_OUT=/tmp NCU_SUMMARY=1
bash scripts/ncu_capture.sh scan_raw k_scan_fast --config cls100 --op scan
ncu -i /tmp/prof_scan_raw.ncu-rep --page source --csv --print-source sass > gpurun_out/src_scan_raw.csv 2>/dev/null
