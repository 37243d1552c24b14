python -m pytest tests -m gpu -x -q 2>&1 | tail -2
B="timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
for r in 1 2; do
$B > gpurun_out/b_pdl_$r.json 2>/dev/null
FSA_PDL=0 $B > gpurun_out/b_nopdl_$r.json 2>/dev/null
done
for f in b_pdl_1 b_nopdl_1 b_pdl_2 b_nopdl_2; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
