#!/bin/bash
# Sweep TMA L2 promotion / cache-policy knobs on the headline config.
for promo in 256 128 64 0; do
  for hint in 0 3 2; do
    MDN_TMA_L2PROMO=$promo MDN_TMA_HINT=$hint timeout 300 python bench.py --steps 30 --warmup 5 \
      --no-cpu-baseline > gpurun_out/knob_p${promo}_h${hint}.log 2>&1
  done
done
