#!/bin/bash
# training wall-time repeat (cls10_c16 read 62 ms in the final sweep vs 36 ms before)
for r in 1 2; do
for cfg in cls10_c16 cls100; do python bench.py --config $cfg --op train --steps 5 --warmup 2 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$cfg', d['value'], d['ms_per_step'])"; done
done
