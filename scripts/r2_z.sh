#!/bin/bash
# k_u8_rows: SUBS=2 A/B and ncu of new vs old fused / encode kernels
mkdir -p gpurun_out/r2z
L='--config image_u8 --steps 100'
echo "== s2 (DP7, ENC DP6, SUBS 2)"
MDN_LIB=libmaddness_s2.so python scripts/bench_lines.py "$L" "$L --mode avg" 2>&1 | cut -c1-150
export NCU_OUT=/tmp NCU_SUMMARY=1
MDN_LIB=libmaddness_dp7.so bash scripts/ncu_capture.sh u8rows_dp7_exact k_u8_rows --config image_u8 -- u8rows_dp6_encode k_u8_rows --config image_u8 --op encode
bash scripts/ncu_capture.sh u8rows_dp6_exact k_u8_rows --config image_u8
MDN_U8_ROWS=0 bash scripts/ncu_capture.sh amm_rt_exact k_amm_rt --config image_u8
for t in u8rows_dp7_exact u8rows_dp6_encode u8rows_dp6_exact amm_rt_exact; do
  ncu -i /tmp/prof_$t.ncu-rep --page source --csv --print-source sass > gpurun_out/r2z/src_$t.csv 2>/dev/null
done
ls -la gpurun_out/r2z
