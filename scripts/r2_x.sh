#!/bin/bash
# full GPU suite + the k_amm_ws lines at the new stage geometry (>= 3 stages)
mkdir -p gpurun_out/r2x
python -m pytest tests -m gpu -q -x > gpurun_out/r2x/pytest.log 2>&1; tail -1 gpurun_out/r2x/pytest.log
for m in 3 4; do
MDN_WS_MINNS=$m python scripts/probe_shapes.py 2>&1 | sed "s/^/M$m /" | cut -c1-160
done
python scripts/bench_lines.py "--config cls10_c64 --steps 100" "--config cls10_c16 --op encode --steps 100" \
  "--config cls10_c32 --op encode --steps 100" "--config cls10_c16 --mode avg --steps 100" \
  "--config scale --mode avg --steps 100" "--config cls10_c32 --mode avg --steps 100" "--config cls10_c64 --mode avg --steps 100"
