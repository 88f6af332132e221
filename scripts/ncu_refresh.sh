#!/bin/bash
# ncu --set full of the dominant kernel of every bench line family (one launch
# each, after a plain run of the same command exited 0), for profiles/rNN/.
#   bash scripts/ncu_refresh.sh   -> gpurun_out/prof_<tag>.ncu-rep
bash scripts/ncu_capture.sh \
  cls100_exact k_amm_ws --config cls100 -- \
  cls100_avg k_amm_ws --config cls100 --mode avg -- \
  cls10_c32_exact k_amm_ws --config cls10_c32 -- \
  scale_exact k_amm_ws --config scale -- \
  tiny_exact k_amm_rt --config tiny -- \
  image_exact k_amm_rt --config image -- \
  image_u8_exact k_u8_rows --config image_u8 -- \
  image_u8_avg k_u8_rows --config image_u8 --mode avg -- \
  cls10_c64_scan_exact k_scan_fast --config cls10_c64 --op scan -- \
  cls100_col_exact k_amm_ws --config cls100 --layout col -- \
  scale_col_exact k_amm_ws --config scale --layout col -- \
  tiny_col_exact k_amm_cm --config tiny --layout col -- \
  image_col_exact k_amm_cm --config image --layout col -- \
  tiny_col_encode_exact k_amm_cm --config tiny --layout col --op encode -- \
  cls100_col_encode_exact k_amm_ws --config cls100 --layout col --op encode -- \
  cls100_encode_exact k_amm_ws --config cls100 --op encode -- \
  image_encode_exact k_amm_rt --config image --op encode -- \
  image_u8_encode_exact k_u8_rows --config image_u8 --op encode -- \
  cls100_scan_exact k_scan_ts --config cls100 --op scan -- \
  image_scan_exact k_scan_fast --config image --op scan -- \
  cls100_encode_pq_exact k_encode_pq --config cls100 --op encode --encoder pq -- \
  scale_encode_pq_exact k_encode_pq --config scale --op encode --encoder pq -- \
  cls10_c16_encode_pq_exact k_encode_pq --config cls10_c16 --op encode --encoder pq -- \
  scale_scan_exact k_scan_fast --config scale --op scan -- \
  cls100_scan_avg k_scan_ts --config cls100 --op scan --mode avg
# the pipeline probe (mdn_amm_probe) of the headline config: same kernel name
# as the fused kernel, told apart by its template arguments
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_amm_ws<float, \(int\)32, \(int\)25, \(int\)0, \(bool\)1, \(bool\)0, \(int\)0, \(bool\)1, \(bool\)0>' -c 1 -f \
    -o ${NCU_OUT:-gpurun_out}/prof_cls100_probe \
    python bench.py --config cls100 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_cls100_probe.log 2>&1
[ -n "$NCU_SUMMARY" ] && python scripts/ncu_summary.py full ${NCU_OUT:-gpurun_out}/prof_cls100_probe.ncu-rep \
    gpurun_out/ncu_full_cls100_probe.json > /dev/null 2>&1
