#!/bin/bash
# A/B: fewest stages (MDN_WS_MINNS) -> larger rows per stage for k_amm_ws
for i in 1 2; do
for m in 4 3 2; do
python scripts/bench_lines.py "MDN_WS_MINNS=$m --config scale --steps 100" "MDN_WS_MINNS=$m --config cls10_c32 --steps 100" \
  "MDN_WS_MINNS=$m --config cls10_c16 --steps 100" "MDN_WS_MINNS=$m --config cls100 --steps 100" \
  "MDN_WS_MINNS=$m --config scale --op encode --steps 100" "MDN_WS_MINNS=$m --config cls10_c64 --op encode --steps 100" \
  "MDN_WS_MINNS=$m --config cls100 --op encode --steps 100" "MDN_WS_MINNS=$m --config cls100 --mode avg --steps 100" 2>&1 | sed "s/^/M$m /"
done
done
