# 128-wide TRSM steps vs 64-wide (FSA_TRSM64=1)
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
for r in 1 2; do
$B > gpurun_out/b106_w$r.json 2>/dev/null
FSA_TRSM64=1 $B > gpurun_out/b106_n$r.json 2>/dev/null
done
for f in w1 n1 w2 n2; do python -c "
import json;d=json.loads(open('gpurun_out/b106_$f.json').read().strip().splitlines()[-1]); t=d['timers_ms']; print('$f', round(d['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['grad'], d['clocks']['sm_mhz'], {k:t[k] for k in ('setup_trsm','setup_fitc','setup_sigma_m')})"; done
