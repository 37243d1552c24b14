timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b56.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b56.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['nll'], [(e['kernel'][:10], round(e['avg_launch_ms'],4), round(e['frac'],3)) for e in d['roofline']['all']])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_oz_reduce -c 5 python tools/spmm_one.py 1 2>&1 | grep -i "duration\|k_oz_reduce" | tail -4
