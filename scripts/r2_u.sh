#!/bin/bash
# A/B: averaging shift-adds as IMAD.HI on the FMA pipe (MDN_AVG_HI = 0 / 2 / 1)
mkdir -p gpurun_out/r2u
run() { local name=$1; shift; timeout 300 python bench.py "$@" --no-cpu-baseline > gpurun_out/r2u/$name.log 2>&1; grep '^{' gpurun_out/r2u/$name.log | tail -1 > gpurun_out/r2u/$name.json; }
for v in base hi2 hi1; do
  if [ $v = base ]; then unset MDN_LIB; else export MDN_LIB=libmaddness_$v.so; fi
  run ${v}_scan_cls100_avg --config cls100 --op scan --mode avg
  run ${v}_col_cls100_avg --config cls100 --mode avg --layout col
  run ${v}_cls100_avg --config cls100 --mode avg
  run ${v}_scan_scale_avg --config scale --op scan --mode avg
  run ${v}_scan_c64_avg --config cls10_c64 --op scan --mode avg
done
python - <<'PY'
import glob, json, os
for f in sorted(glob.glob("gpurun_out/r2u/*.json")):
    try: d = json.loads(open(f).read())
    except Exception: print(os.path.basename(f), "ERR"); continue
    r = d.get("roofline") or {}
    print(os.path.basename(f)[:-5], "%.3e" % d.get("value", 0), "frac=%.3f" % r.get("frac", 0), (d.get("parity") or {}).get("ok"))
PY
