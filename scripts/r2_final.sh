#!/bin/bash
# round-2 final evidence: GPU suite + smoke, the bench sweep, then the ncu refresh
mkdir -p gpurun_out/r2final
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r2final/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2final/gputest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2final/smoke.log
rm -rf gpurun_out/final; bash scripts/bench_final.sh > gpurun_out/final_summary.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/r2final/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2final/ncu_launch.log 2>&1
python scripts/ncu_summary.py launches gpurun_out/r2final/launches.csv gpurun_out/r2final/launches.json > /dev/null 2>&1
rm -f gpurun_out/ncu_full_*.json
NCU_OUT=/tmp NCU_SUMMARY=1 bash scripts/ncu_refresh.sh > gpurun_out/ncu_refresh.log 2>&1
tail -3 gpurun_out/r2final/gputest.log
