# session-4 state check: GPU suite, smoke, default bench line
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['value'], d['e2e'], d['clocks'], d['roofline'].get('frac')); print(d.get('timers_ms'))"
