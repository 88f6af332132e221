set -e
mkdir -p gpurun_out
for cfg in image_u8 image; do
python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_$cfg.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_amm_ws -s 1 -c 1 -o gpurun_out/prof_$cfg python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_$cfg.log 2>&1
done
