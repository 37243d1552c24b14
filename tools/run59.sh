for w in 1 2 3 4 6; do FSA_SYRK_WAVES=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b59.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b59.json').read().strip().splitlines()[-1]); print('waves $w', round(d['ms_per_step'],3), d['timers_ms']['setup_fitc_syrk'], d['timers_ms']['setup_fitc'])"; done
