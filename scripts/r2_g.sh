#!/bin/bash
# full GPU suite + default bench + launch list + headline ncu
mkdir -p gpurun_out/r2g
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r2g/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2g/gputest.log
timeout 600 python bench.py > gpurun_out/r2g/default.json 2> gpurun_out/r2g/default.err
echo "bench rc=$?" >> gpurun_out/r2g/default.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/r2g/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2g/ncu_launch.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/r2g/launches.csv gpurun_out/r2g/launches.json > /dev/null 2>&1
NCU_OUT=gpurun_out/r2g NCU_SUMMARY=1 bash scripts/ncu_capture.sh cls100_exact k_amm_ws --config cls100 -- cls100_probe 'k_amm_ws<float,.32,.25,.0,.true,.false,.0,.true>' --config cls100 > gpurun_out/r2g/ncu_cap.log 2>&1
tail -3 gpurun_out/r2g/gputest.log
