#!/bin/bash
# the four captures the refresh missed (kernel renamed / template widened)
export NCU_OUT=/tmp NCU_SUMMARY=1
bash scripts/ncu_capture.sh image_u8_exact k_u8_rows --config image_u8 -- image_u8_avg k_u8_rows --config image_u8 --mode avg -- image_u8_encode_exact k_u8_rows --config image_u8 --op encode
sed -n '/pipeline probe/,$p' scripts/ncu_refresh.sh > /tmp/probe.sh; bash /tmp/probe.sh
ls gpurun_out/ncu_full_image_u8* gpurun_out/ncu_full_cls100_probe.json
