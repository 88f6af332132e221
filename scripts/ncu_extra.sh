#!/bin/bash
mkdir -p gpurun_out
run() {  # tag, kernel regex, bench args...
  local tag=$1; local kre=$2; shift 2
  python bench.py "$@" --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 || { echo "plain $tag failed"; return; }
  ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o gpurun_out/prof_$tag \
      python bench.py "$@" --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
}
run pq_encode_cls100 k_encode_pq --config cls100 --op encode --encoder pq
run scale_col_exact k_amm_cm --config scale --layout col
run cls100_encode_col k_amm_cm --config cls100 --layout col --op encode
