# knob sweep on the current build: SYRK split variants, SpMM epilogue prefetch distance
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
run() { env $1 $B > gpurun_out/b111.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b111.json').read().strip().splitlines()[-1]); t=d['timers_ms']; print('$1', round(d['ms_per_step'],3), round(d['pcg_ms'],3), d['clocks']['sm_mhz'], {k:t[k] for k in ('setup_fitc_syrk','spmm','setup_fitc')})"; }
run X=0
run FSA_GEMM_REDUCE=0
run FSA_GEMM_REDUCE=2
run FSA_SPMM_EPF=2
run FSA_SPMM_EPF=6
run FSA_SPMM_EPF=8
run FSA_SPMM_EPF=0
run X=1
