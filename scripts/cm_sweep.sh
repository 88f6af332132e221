for R in 256 128 64 32; do for cfg in cls100 scale; do
MDN_CM_R=$R timeout 300 python bench.py --layout col --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cmr.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/cmr.log').read().strip().splitlines()[-1]);print('R=$R $cfg', '%.3e'%d['value'])" 2>&1 | tail -1
done; done
for cfg in cls100 scale; do
MDN_CM_SIMPLE=1 timeout 300 python bench.py --layout col --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cmr.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/cmr.log').read().strip().splitlines()[-1]);print('simple $cfg', '%.3e'%d['value'])" 2>&1 | tail -1
done
