# Sigma_mn on the side stream under the Sigma_m Cholesky panels
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm > gpurun_out/b98_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/b98_$r.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['clocks']['sm_mhz'], d['timers_ms'])"; done
FSA_SERIAL_CROSS_COV=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm > gpurun_out/b98_s.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/b98_s.json').read().strip().splitlines()[-1]); print('serial', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['clocks']['sm_mhz'])"
