#!/bin/bash
mkdir -p gpurun_out/r2u
python -m pytest tests/test_gpu_u8.py tests/test_gpu_small.py tests/test_gpu_edges.py -m gpu -q -x > gpurun_out/r2u/pytest.log 2>&1; tail -1 gpurun_out/r2u/pytest.log
python scripts/bench_lines.py "--config image_u8 --steps 100" "--config image_u8 --mode avg --steps 100" \
  "--config image --steps 100" "--config tiny --steps 100" "--config image --mode avg --steps 100"
