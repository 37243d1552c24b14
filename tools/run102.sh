# L2 residency hints of the sweep kernels: A/B against the nohints library (FSA_LIB), same box, alternating
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
for r in 1 2 3; do
$B > gpurun_out/b102_h$r.json 2>/dev/null
FSA_LIB=$PWD/build/nohints/libfsa_b200.so $B > gpurun_out/b102_n$r.json 2>/dev/null
done
for f in h1 n1 h2 n2 h3 n3; do python -c "
import json;d=json.loads(open('gpurun_out/b102_$f.json').read().strip().splitlines()[-1]); t=d['timers_ms']; print('$f', round(d['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['clocks']['sm_mhz'], {k:t[k] for k in ('cg_blas1','spmm','lowrank_project','lowrank_expand')})"; done
