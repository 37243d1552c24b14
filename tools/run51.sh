# projection: 8 slicer warps inside the GEMM (FSA_OZ_SLICE=1) vs the separate slicing kernel
for v in "FSA_OZ_SLICE=0" "FSA_OZ_SLICE=1"; do env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b51.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b51.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), d['nll'], [(e['kernel'][:10], round(e['avg_launch_ms'],4), round(e['frac'],3)) for e in d['roofline']['all']])"; done
FSA_OZ_SLICE=1 timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -2
