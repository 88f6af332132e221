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
  image_u8_exact k_amm_rt --config image_u8 -- \
  cls100_col_exact k_amm_ws --config cls100 --layout col -- \
  scale_col_exact k_amm_ws --config scale --layout col -- \
  tiny_col_exact k_amm_cm --config tiny --layout col -- \
  image_col_exact k_amm_cm --config image --layout col -- \
  tiny_col_encode_exact k_amm_cm --config tiny --layout col --op encode -- \
  cls100_col_encode_exact k_amm_ws --config cls100 --layout col --op encode -- \
  cls100_encode_exact k_amm_ws --config cls100 --op encode -- \
  image_encode_exact k_amm_rt --config image --op encode -- \
  image_u8_encode_exact k_amm_rt --config image_u8 --op encode -- \
  cls100_scan_exact k_scan_fast --config cls100 --op scan -- \
  image_scan_exact k_scan_fast --config image --op scan -- \
  cls100_encode_pq_exact k_encode_pq --config cls100 --op encode --encoder pq
