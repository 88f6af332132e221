#!/bin/bash
# k_u8_rows with one flat chunk loop (no constant re-reads at SUBS = 2): parity, lines, avg variants, ncu
mkdir -p gpurun_out/r2y
timeout 900 python -m pytest tests/test_gpu_u8.py tests/test_gpu_u8_rows.py tests/test_gpu_small.py tests/test_gpu_edges.py -m gpu -q -x > gpurun_out/r2y/pytest.log 2>&1; tail -1 gpurun_out/r2y/pytest.log
L='--config image_u8 --steps 100'
python scripts/bench_lines.py "$L" "$L --mode avg" "$L --op encode" 2>&1 | cut -c1-150
for v in a26 a27; do echo "== $v"; MDN_LIB=libmaddness_$v.so python scripts/bench_lines.py "$L --mode avg" 2>&1 | cut -c1-150; done
python scripts/bench_lines.py "$L" "$L --mode avg" "$L --op encode" 2>&1 | cut -c1-150
export NCU_OUT=/tmp NCU_SUMMARY=1
bash scripts/ncu_capture.sh u8r_exact k_u8_rows --config image_u8 -- u8r_encode k_u8_rows --config image_u8 --op encode
