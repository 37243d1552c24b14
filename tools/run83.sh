# session-3 baseline: GPU suite, smoke, config-2 bench
timeout 1200 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b83.json 2> gpurun_out/b83.err; echo c2=$?
python -c "
import json;d=json.loads(open('gpurun_out/b83.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['value'], d['e2e']['value'], d['clocks']); print(json.dumps(d['roofline'])[:1500])"
