timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b77.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b77.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['nll'], d['grad'], d['clocks']['sm_mhz'])"; done
