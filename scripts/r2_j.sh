#!/bin/bash
mkdir -p gpurun_out/r2j
python bench.py --config cls100 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2j/plain.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:k_amm_ws<float, \(int\)32, \(int\)25, \(int\)0, \(bool\)1, \(bool\)0, \(int\)0, \(bool\)1>' -c 1 -f \
    -o /tmp/prof_cls100_probe \
    python bench.py --config cls100 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2j/ncu_probe.log 2>&1
python scripts/ncu_summary.py full /tmp/prof_cls100_probe.ncu-rep gpurun_out/r2j/ncu_full_cls100_probe.json > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r2j/gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2j/gputest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2j/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2j/smoke.log
tail -3 gpurun_out/r2j/gputest.log
