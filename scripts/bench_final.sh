#!/bin/bash
# Every bench line of DESIGN.md §6 with the current code (1 GPU), into gpurun_out/final/.
mkdir -p gpurun_out/final
run() {  # name, args...
  local name=$1; shift
  timeout 600 python bench.py "$@" > gpurun_out/final/$name.log 2>&1 || echo "FAILED $name" >> gpurun_out/final/failed.txt
  grep '^{' gpurun_out/final/$name.log | tail -1 > gpurun_out/final/$name.json
}
run default
for cfg in cls100 cls10_c16 cls10_c32 cls10_c64 scale tiny image image_u8; do
  for mode in exact avg; do run ${cfg}_${mode} --config $cfg --mode $mode --no-cpu-baseline; done
done
for cfg in cls100 scale cls10_c16 tiny image; do
  for mode in exact avg; do run col_${cfg}_${mode} --config $cfg --mode $mode --layout col --no-cpu-baseline; done
done
for cfg in cls100 cls10_c16 cls10_c32 cls10_c64 scale tiny image; do
  run encode_${cfg} --config $cfg --op encode --no-cpu-baseline
  run scan_${cfg} --config $cfg --op scan --no-cpu-baseline
done
run encode_image_u8 --config image_u8 --op encode --no-cpu-baseline
run scan_cls100_avg --config cls100 --op scan --mode avg --no-cpu-baseline
for cfg in cls100 scale cls10_c16 tiny image; do run encode_col_${cfg} --config $cfg --op encode --layout col --no-cpu-baseline; done
for cfg in cls100 cls10_c16 scale tiny; do run pq_encode_${cfg} --config $cfg --op encode --encoder pq --no-cpu-baseline; done
run pq_amm_cls100 --config cls100 --encoder pq --no-cpu-baseline
run scale_strong --config scale --strong --no-cpu-baseline
for cfg in tiny cls10_c16 cls100 scale image; do run train_${cfg} --config $cfg --op train --steps 3 --warmup 1 --cpu-seconds 5; done
run reference --impl reference --steps 3 --warmup 3
MDN_DIST_BACKEND=gloo run gloo2_functional --gpus 2 --steps 20 --config cls100 --cpu-seconds 2
python - <<'PY'
import glob, json, os
for f in sorted(glob.glob("gpurun_out/final/*.json")):
    try:
        d = json.loads(open(f).read())
    except Exception:
        print(os.path.basename(f), "ERR"); continue
    r = d.get("roofline") or {}
    print(os.path.basename(f)[:-5], "%.3e %s" % (d.get("value", 0), d.get("unit", "")),
          "frac=%.3f" % r["frac"] if r.get("frac") is not None else "", (d.get("parity") or {}).get("ok"))
PY
