# one-barrier potrf diagonal block: parity + timing
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/b82.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b82.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), repr(d['nll']), d['clocks']['sm_mhz'])"; done
timeout 900 ncu --nvtx --nvtx-include "one_eval/" --metrics gpu__time_duration.sum --clock-control none -k regex:k_potrf --csv --log-file gpurun_out/potrf82.csv python tools/one_eval.py > /dev/null 2>&1; echo ncu=$?
python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/potrf82.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
from collections import defaultdict
t=defaultdict(list)
for r in rows[1:]:
    try: t[r[ki][:40]].append(float(r[vi].replace(',','')))
    except: pass
for k,v in t.items(): print(k, len(v), round(sum(v)/1e3/3,1), 'us per eval')
P
