# k_xr_planes at 256 threads, 4 CTAs per SM (37 clusters of 8 in one wave)
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/one_eval.py 2>&1 | tail -2
for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b90_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/b90_$r.json').read().strip().splitlines()[-1]); a={x['kernel'][:12]:round(x['avg_launch_ms']*1e3,1) for x in d['roofline']['all']}; print(round(d['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['clocks']['sm_mhz'], a, d['timers_ms'].get('cg_blas1'))"; done
timeout 600 ncu --nvtx --nvtx-include "one_eval/" --metrics gpu__time_duration.sum --clock-control none -k regex:"k_xr|k_oz_reduce|k_colsum|k_oz_planes|k_oz_gemm" --csv --log-file gpurun_out/small90.csv python tools/one_eval.py > /dev/null 2>&1; echo ncu=$?
python - <<'P'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/small90.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
t=defaultdict(list)
for r in rows[1:]:
    try: t[r[ki][:40]].append(float(r[vi].replace(',','')))
    except: pass
for k,v in t.items(): print(k, len(v), round(sum(v)/len(v)/1e3,2), 'us avg')
P
