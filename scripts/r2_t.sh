#!/bin/bash
# ncu --set full of the kernels changed in round 2 session 2 (dp4a byte trees, scan launch bounds)
NCU_OUT=/tmp NCU_SUMMARY=1 bash scripts/ncu_capture.sh \
  image_u8_exact k_amm_rt --config image_u8 -- \
  image_u8_avg k_amm_rt --config image_u8 --mode avg -- \
  image_u8_encode_exact k_amm_rt --config image_u8 --op encode -- \
  cls100_scan_exact k_scan_fast --config cls100 --op scan -- \
  cls10_c64_scan_exact k_scan_fast --config cls10_c64 --op scan
