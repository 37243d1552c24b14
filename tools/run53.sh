# balanced base-256 digits (7 planes, 34 products)
timeout 600 python -m pytest tests/test_gpu_ozaki.py -q -x --timeout 300 -p no:cacheprovider -s 2>&1 | grep -v "^$" | tail -12
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -4
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b53.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b53.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['nll'], [(e['kernel'][:10], round(e['avg_launch_ms'],4), round(e['frac'],3)) for e in d['roofline']['all']])"
