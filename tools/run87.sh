# pair path with 8-aligned B tiles (N = 40, 120 on M = 128 kind::i8): legality + accuracy + config-4 timing
export FSA_OZ_PAIR_NC8=1
timeout 300 python -m pytest tests/test_gpu_ozaki.py -q -s -k pair -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_sharded.py -q -k 72 -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/c4_87.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/c4_87.json').read().strip().splitlines()[-1]); a={x['kernel'][:12]:round(x['avg_launch_ms']*1e3,1) for x in d['roofline']['all']}; print('c4 nc8', round(d['ms_per_step'],3), repr(d['nll']), d['clocks']['sm_mhz'], a)"
