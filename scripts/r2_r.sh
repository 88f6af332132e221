#!/bin/bash
# Round 2 (session 2) A/B: 8-bit byte tree in the dp4a form (MDN_BQ_DP bitmask)
# and the standalone scan's launch bounds (MDN_SCAN_MINB).
mkdir -p gpurun_out/r2r
B="--no-cpu-baseline --parity-rows 4096 --steps 100"
for i in 1 2; do
for v in main dp7 dp6 dp4 dp1; do
  L=libmaddness.so; [ $v != main ] && L=libmaddness_$v.so
  [ -f paper_2106_10860_b200/$L ] || continue
  MDN_LIB=$L timeout 300 python bench.py --config image_u8 $B > gpurun_out/r2r/u8_${v}_$i.json 2>&1
  MDN_LIB=$L timeout 300 python bench.py --config image_u8 --op encode $B > gpurun_out/r2r/u8enc_${v}_$i.json 2>&1
done
for v in main mb1; do
  L=libmaddness.so; [ $v != main ] && L=libmaddness_$v.so
  [ -f paper_2106_10860_b200/$L ] || continue
  for c in cls100 scale cls10_c16 cls10_c64 image tiny; do
    MDN_LIB=$L timeout 300 python bench.py --config $c --op scan $B > gpurun_out/r2r/scan_${c}_${v}_$i.json 2>&1
  done
done
done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob('gpurun_out/r2r/*.json')):
    try:
        d=json.loads(open(f).read().strip().split('\n')[-1])
        print(os.path.basename(f), '%.4e'%d['value'], d['parity']['ok'], round(d['roofline']['frac'],3))
    except Exception as e:
        print(os.path.basename(f), 'ERR', open(f).read()[-300:])
PY
