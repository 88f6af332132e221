#!/bin/bash
# column-major fused cls100: scanner parts by TMA tensor stores (MDN_CM_TSTORE) vs LDS + STG readback;
# headline unchanged by the extra kernel parameter; ncu of k_scan_ts kept for the summary
echo "== tests default"; timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
echo "== tests cts1"; MDN_LIB=libmaddness_cts1.so timeout 900 python -m pytest tests/test_gpu_colmajor.py tests/test_gpu_edges.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1
LINES=("--config cls100 --layout col --steps 100" "--config cls100 --layout col --mode avg --steps 100" "--config cls100 --steps 100")
for v in "" cts1 "" cts1; do
  lib=libmaddness.so; [ -n "$v" ] && lib=libmaddness_$v.so
  echo "== $lib"
  MDN_LIB=$lib python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
done
NCU_OUT=gpurun_out bash scripts/ncu_capture.sh scan_ts k_scan_ts --config cls100 --op scan
python scripts/ncu_summary.py full gpurun_out/prof_scan_ts.ncu-rep gpurun_out/ncu_full_scan_ts.json 2>&1 | tail -3
ncu -i gpurun_out/prof_scan_ts.ncu-rep --page raw --csv 2>&1 | head -c 600
