#!/bin/bash
# Round 2 (session 2): GPU tests + the lines touched by the dp4a byte trees and the scan launch bounds.
mkdir -p gpurun_out/r2s
python -m pytest tests -m gpu -q -x > gpurun_out/r2s/pytest_gpu.log 2>&1; tail -2 gpurun_out/r2s/pytest_gpu.log
python scripts/bench_lines.py "--config image_u8 --steps 100" "--config image_u8 --op encode --steps 100" \
  "--config image_u8 --mode avg --steps 100" "--config cls100 --op scan --steps 100" \
  "--config cls10_c64 --op scan --steps 100" "--config scale --op scan --steps 100" \
  "--config image --op scan --steps 100" "--config cls100 --steps 100" > gpurun_out/r2s/lines.txt 2>&1
cat gpurun_out/r2s/lines.txt
