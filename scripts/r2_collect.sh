#!/bin/bash
# copy the evidence of scripts/r2_final.sh from gpurun_out/ into profiles/r02/
set -e
mkdir -p profiles/r02/bench_final
cp gpurun_out/final/*.json profiles/r02/bench_final/ 2>/dev/null || true
cp gpurun_out/final_summary.txt profiles/r02/bench_final/SUMMARY.txt 2>/dev/null || true
[ -f gpurun_out/final/failed.txt ] && cp gpurun_out/final/failed.txt profiles/r02/bench_final/ || true
cp gpurun_out/ncu_full_*.json profiles/r02/ 2>/dev/null || true
cp gpurun_out/r2final/launches.csv profiles/r02/ncu_launches_bench.csv 2>/dev/null || true
cp gpurun_out/r2final/launches.json profiles/r02/ncu_launches_bench.json 2>/dev/null || true
cp gpurun_out/r2final/gputest.log profiles/r02/gputest_final.log 2>/dev/null || true
cp gpurun_out/r2final/smoke.log profiles/r02/smoke_final.log 2>/dev/null || true
python scripts/traffic_from_summaries.py profiles/r02 > /dev/null
tail -3 profiles/r02/gputest_final.log; tail -2 profiles/r02/smoke_final.log
