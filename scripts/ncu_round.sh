#!/bin/bash
# ncu --set full of the top kernel for several bench configs (each after a plain run).
mkdir -p gpurun_out
run() {  # tag, bench args...
  local tag=$1; shift
  python bench.py "$@" --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$tag.log 2>&1 || { echo "plain $tag failed"; return; }
  ncu --set full --clock-control none --import-source on -k regex:k_amm -s 1 -c 1 -o gpurun_out/prof_$tag \
      python bench.py "$@" --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$tag.log 2>&1
}
run image_u8_exact --config image_u8
run image_exact --config image
run tiny_exact --config tiny
run cls100_col_exact --config cls100 --layout col
run cls100_avg --config cls100 --mode avg
