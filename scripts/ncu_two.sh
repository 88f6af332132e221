#!/bin/bash
mkdir -p gpurun_out
run() {  # tag, bench args...
  local tag=$1; shift
  python bench.py "$@" --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 || { echo "plain $tag failed"; return; }
  ncu --set full --clock-control none --import-source on -k regex:k_amm -s 1 -c 1 -o gpurun_out/prof_$tag \
      python bench.py "$@" --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
}
run scale_exact --config scale
run cls10_c32_exact --config cls10_c32
