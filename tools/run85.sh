# expansion weights 2..8 (FSA_OZ_EXP_W8=1) accuracy + timing; config-4 A/B of the projection weights
export FSA_OZ_EXP_W8=1
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -s -p no:cacheprovider 2>&1 | grep -E "ozaki-dmma|passed|failed|Error|assert" | head -20
timeout 900 python -m pytest tests/test_gpu_configs.py -q -p no:cacheprovider 2>&1 | tail -2
unset FSA_OZ_EXP_W8
for r in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export FSA_OZ_EXP_W8=1; else unset FSA_OZ_EXP_W8; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/ab85_${v}_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab85_${v}_$r.json').read().strip().splitlines()[-1]); a={x['kernel'][:12]:round(x['avg_launch_ms']*1e3,1) for x in d['roofline']['all']}; print('expw8=$v', round(d['ms_per_step'],3), repr(d['nll']), d['clocks']['sm_mhz'], a)"
done; done
unset FSA_OZ_EXP_W8
for v in 1 0 2; do
  unset FSA_OZ_PROJ_W9 FSA_OZ_EXP_W8
  if [ $v = 1 ]; then export FSA_OZ_PROJ_W9=1; fi
  if [ $v = 2 ]; then export FSA_OZ_EXP_W8=1; fi
  timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/ab85_c4_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab85_c4_$v.json').read().strip().splitlines()[-1]); a={x['kernel'][:12]:round(x['avg_launch_ms']*1e3,1) for x in d['roofline']['all']}; print('c4 v=$v', round(d['ms_per_step'],3), repr(d['nll']), d['clocks']['sm_mhz'], a)"
done
