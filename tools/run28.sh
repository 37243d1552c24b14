timeout 120 python tools/spmm_attr.py 2>&1 | tail -2
python -m pytest tests/test_gpu_ozaki.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
$B > gpurun_out/b_now.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b_now.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), [(e['kernel'][:10], round(e['avg_launch_ms'],4), round(e['frac'],3)) for e in d['roofline']['all']])"
