timeout 600 python tools/probe_cmp.py
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -2
for v in "FSA_HOST_PROBES=1" "FSA_X=0"; do env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 4 > gpurun_out/b78.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b78.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), d['nll'], d['clocks']['sm_mhz'])"; done
