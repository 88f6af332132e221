#!/bin/bash
# staged scan: FMA-pipe share of the odd-lane adds (MIX 0 = ALU, 3 = 2 of 3 words IMAD, k64 ~ all IMAD, k2 = half)
LINES=("--config cls100 --op scan --steps 100" "--config cls100 --op scan --mode avg --steps 100")
python scripts/bench_lines.py "${LINES[@]}" 2>&1 | cut -c1-150
echo "== MIX 3"; MDN_SCAN_MIX=3 python scripts/bench_lines.py "${LINES[0]}" 2>&1 | cut -c1-150
for v in k2 k64; do echo "== $v MIX forced"; MDN_SCAN_MIX=3 MDN_LIB=libmaddness_$v.so python scripts/bench_lines.py "${LINES[0]}" 2>&1 | cut -c1-150; done
