# full GPU suite + smoke with the lean SpMM (k_spmm_v3), then the config-2 bench
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for v in "FSA_SPMM=rt" "FSA_SPMM_EPB=1"; do env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b38.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b38.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), round(d['sweep']['t_measured_ms'] if 'sweep' in d else 0,4), [(e['kernel'][:10], round(e['avg_launch_ms'],4), round(e['frac'],3)) for e in d['roofline']['all']])"; done
