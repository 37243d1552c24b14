TAG=lean-epi FLAGS=0 python tools/spmm_ab.py
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b42.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b42.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), [(e['kernel'][:10], round(e['avg_launch_ms'],4), round(e['frac'],3)) for e in d['roofline']['all']])"
