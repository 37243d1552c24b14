# default bench line (20 steps) for the record + reference arm
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 300 python tools/one_eval.py 2>&1 | tail -3
python -c "
import json;d=json.loads(open('gpurun_out/bench_c2.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e'], d['clocks'], d['steps']); print([ (r['kernel'][:12], round(r['avg_launch_ms'],4), round(r['frac'],3), r['traffic']) for r in d['roofline']['all']]); print(d['roofline']['sweep']['own_floor'])"
