# projection weights 2..8 (28 products) vs 2..9 (FSA_OZ_PROJ_W9=1): accuracy + config-2 parity + timing
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -s -p no:cacheprovider 2>&1 | grep -E "ozaki-dmma|passed|failed|Error" | head -20
timeout 900 python -m pytest tests/test_gpu_configs.py -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export FSA_OZ_PROJ_W9=1; else unset FSA_OZ_PROJ_W9; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/ab84_${v}_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab84_${v}_$r.json').read().strip().splitlines()[-1]); a={x['kernel'][:12]:round(x['avg_launch_ms']*1e3,1) for x in d['roofline']['all']}; print('w9=$v', round(d['ms_per_step'],3), repr(d['nll']), d['clocks']['sm_mhz'], a)"
done; done
