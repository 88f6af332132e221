for S in 0 1; do for cfg in cls100 scale; do
MDN_CM_SIMPLE=$S timeout 300 python bench.py --layout col --op encode --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cmr.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/cmr.log').read().strip().splitlines()[-1]);print('encode simple=$S $cfg', '%.3e'%d['value'], '%.3f'%d['roofline']['frac'])" 2>&1 | tail -1
done; done
