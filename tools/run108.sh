# wide expansion passes with the column tiles looped inside each point tile (k_oz_expand<MULTI>)
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b108_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/b108_$r.json').read().strip().splitlines()[-1]); t=d['timers_ms']; print(round(d['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['grad'], d['clocks']['sm_mhz'])"; done
timeout 600 ncu --nvtx --nvtx-include "one_eval/" --metrics gpu__time_duration.sum --clock-control none -k regex:"k_oz_expand|k_oz_wexp|k_oz_planes_w|k_sum_tiles" --csv --log-file gpurun_out/small108.csv python tools/one_eval.py > /dev/null 2>&1; echo ncu=$?
python - <<'P'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/small108.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
t=defaultdict(list)
for r in rows[1:]:
    try: t[r[ki][:60]].append(float(r[vi].replace(',','')))
    except: pass
for k,v in t.items(): print(k, len(v), round(sum(v)/len(v)/1e3,2), 'us avg', round(sum(v)/3e3,1), 'us per eval')
P
