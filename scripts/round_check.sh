#!/bin/bash
# Round checkpoint: full GPU tests, smoke, default bench, reference arm, launch list + full ncu of the headline kernel.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_launch.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
CMD2="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD2 > gpurun_out/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_amm -s 1 -c 1 -f -o /tmp/prof_cls100_exact $CMD2 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
python scripts/ncu_summary.py full /tmp/prof_cls100_exact.ncu-rep gpurun_out/ncu_full_cls100_exact_check.json > /dev/null 2>&1
