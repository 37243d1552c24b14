timeout 300 python tools/spmm_attr.py > gpurun_out/spmm_attr_pr.log 2>&1; head -5 gpurun_out/spmm_attr_pr.log
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
for r in 1 2; do
$B > gpurun_out/b_pr_$r.json 2>/dev/null
FSA_SPMM_KERNEL=rt $B > gpurun_out/b_rt_$r.json 2>/dev/null
done
for f in b_pr_1 b_rt_1 b_pr_2 b_rt_2; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); r=d['roofline']['all'][0]; print('$f', round(d['ms_per_step'],3), round(r['avg_launch_ms'],4), round(r['frac'],3), d['clocks']['sm_mhz'])"; done
