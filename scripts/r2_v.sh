#!/bin/bash
# A/B: rows per stage of k_amm_ws (MDN_WS_RMAX) with the stage ring cap raised to 16
mkdir -p gpurun_out/r2v
python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2v/pytest.log 2>&1; tail -1 gpurun_out/r2v/pytest.log
for i in 1 2; do
for r in 256 16 8; do
python scripts/bench_lines.py "MDN_WS_RMAX=$r --config scale --steps 100" "MDN_WS_RMAX=$r --config cls10_c32 --steps 100" \
  "MDN_WS_RMAX=$r --config cls10_c64 --steps 100" "MDN_WS_RMAX=$r --config cls100 --steps 100" \
  "MDN_WS_RMAX=$r --config scale --op encode --steps 100" "MDN_WS_RMAX=$r --config cls10_c64 --op encode --steps 100" \
  "MDN_WS_RMAX=$r --config cls100 --mode avg --steps 100" 2>&1 | sed "s/^/R$r /"
done
done
