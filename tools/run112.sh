# split-K reduce + core solve + W slicing in one launch (k_core_fused) vs the three kernels (FSA_NO_CORE_FUSE=1)
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
for r in 1 2 3; do
$B > gpurun_out/b112_f$r.json 2>/dev/null
FSA_NO_CORE_FUSE=1 $B > gpurun_out/b112_n$r.json 2>/dev/null
done
for f in f1 n1 f2 n2 f3 n3; do python -c "
import json;d=json.loads(open('gpurun_out/b112_$f.json').read().strip().splitlines()[-1]); t=d['timers_ms']; print('$f', round(d['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['clocks']['sm_mhz'], {k:t[k] for k in ('core_solve','lowrank_project','lowrank_expand')})"; done
