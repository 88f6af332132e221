#!/bin/bash
# A/B of the 3-instruction averaging tree (MDN_AVG_LEA): the averaging parity tests, then the avg lines
mkdir -p gpurun_out/r2t
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r2t/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2t/gputest.log
run() { local name=$1; shift; timeout 300 python bench.py "$@" --no-cpu-baseline > gpurun_out/r2t/$name.log 2>&1; grep '^{' gpurun_out/r2t/$name.log | tail -1 > gpurun_out/r2t/$name.json; }
run scan_cls100_avg --config cls100 --op scan --mode avg
run col_cls100_avg --config cls100 --mode avg --layout col
run cls100_avg --config cls100 --mode avg
run scale_avg --config scale --mode avg
run col_scale_avg --config scale --mode avg --layout col
run cls10_c64_avg --config cls10_c64 --mode avg
run col_cls10_c16_avg --config cls10_c16 --mode avg --layout col
run default
python - <<'PY'
import glob, json, os
for f in sorted(glob.glob("gpurun_out/r2t/*.json")):
    try: d = json.loads(open(f).read())
    except Exception: print(os.path.basename(f), "ERR"); continue
    r = d.get("roofline") or {}
    print(os.path.basename(f)[:-5], "%.3e" % d.get("value", 0), "frac=%.3f" % r.get("frac", 0), (d.get("parity") or {}).get("ok"))
PY
tail -3 gpurun_out/r2t/gputest.log
# ncu of the lines whose kernels changed
rm -f gpurun_out/ncu_full_*.json
NCU_OUT=/tmp NCU_SUMMARY=1 bash scripts/ncu_capture.sh \
  cls100_avg k_amm_ws --config cls100 --mode avg -- \
  cls100_scan_avg k_scan_ts --config cls100 --op scan --mode avg > gpurun_out/r2t/ncu.log 2>&1
ls gpurun_out/ncu_full_*.json
