#!/bin/bash
# k_u8_rows with per-mode (SUBS, DP): u8 parity suites, then the three image_u8 lines twice
mkdir -p gpurun_out/r2y
timeout 900 python -m pytest tests/test_gpu_u8.py tests/test_gpu_u8_rows.py tests/test_gpu_small.py tests/test_gpu_edges.py -m gpu -q -x > gpurun_out/r2y/pytest.log 2>&1; tail -1 gpurun_out/r2y/pytest.log
L='--config image_u8 --steps 100'
for r in 1 2; do
  python scripts/bench_lines.py "$L" "$L --mode avg" "$L --op encode" 2>&1 | cut -c1-150
done
echo "== old k_amm_rt"
MDN_U8_ROWS=0 python scripts/bench_lines.py "$L" "$L --mode avg" "$L --op encode" 2>&1 | cut -c1-150
