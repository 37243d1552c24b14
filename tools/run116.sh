# final check of the committed tree: GPU suite, smoke, default bench line
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e']['value'], d['e2e']['ms_per_step'], d['clocks'], d['steps'], d['gpu_launches']); print([(r['kernel'][:10], round(r['frac'],3), r['traffic']) for r in d['roofline']['all']])"
