# SpMM A/B: round-1 kernel vs metadata-in-smem ring of depth 2/3/4
FSA_SPMM=rt TAG=rt FLAGS=0,15,3 python tools/spmm_ab.py
for ns in 2 3 4; do FSA_SPMM_NS=$ns TAG=ms$ns FLAGS=0,15,3,2 python tools/spmm_ab.py; done
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
for v in "FSA_SPMM=rt" "FSA_SPMM_NS=3"; do env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b31.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b31.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), [(e['kernel'][:10], round(e['avg_launch_ms'],4), round(e['frac'],3)) for e in d['roofline']['all']])"; done
