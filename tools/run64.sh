for i in 1 2; do for v in "FSA_T_DMMA=1" "FSA_X=0"; do env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b64.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b64.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"; done; done
