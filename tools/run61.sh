timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b61.json 2> gpurun_out/b61.err; echo c4=$?
python -c "
import json;d=json.loads(open('gpurun_out/b61.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['value'], d['clocks'], [(e['kernel'][:14], round(e['avg_launch_ms'],4), round(e['frac'],3), round(e['share_of_step'],3)) for e in d['roofline']['all']], d['roofline']['sweep']['t_measured_ms'], d['timers_ms'])"
