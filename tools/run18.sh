python -m pytest tests/test_gpu_ozaki.py tests/test_cpp_shim.py tests/test_fsagp_facade.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b_c4.json 2> gpurun_out/b_c4.err; echo c4_rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/b_c4.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['ms_per_step'],1), 'prof', round(r['profiled_pass_ms_per_step'],1), [ (e['kernel'][:14], round(e['avg_launch_ms'],3), round(e['frac'],3)) for e in r['all']], d['sweeps'], d['clocks'])
print(d['timers_ms'])"
