# L2 residency schemes (FSA_L2_MODE bit masks, bulk.cuh): default build = 63, variants via FSA_LIB
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
for r in 1 2; do
$B > gpurun_out/b103_63_$r.json 2>/dev/null
for m in 0 1 33 35 47 55; do FSA_LIB=$PWD/build/l2mode$m/libfsa_b200.so $B > gpurun_out/b103_${m}_$r.json 2>/dev/null; done
done
for r in 1 2; do for m in 0 1 33 35 47 55 63; do python -c "
import json;d=json.loads(open('gpurun_out/b103_${m}_$r.json').read().strip().splitlines()[-1]); t=d['timers_ms']; print('mode $m', round(d['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['clocks']['sm_mhz'], {k:t[k] for k in ('cg_blas1','spmm','lowrank_project','lowrank_expand')})"; done; done
