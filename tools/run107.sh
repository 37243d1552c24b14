# k_block_gram at 4 resident CTAs (64 registers); dgemm expand tile variants under the 128-wide TRSM
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "parity or configs" 2>&1 | tail -2
timeout 600 ncu --nvtx --nvtx-include "one_eval/" --metrics gpu__time_duration.sum --clock-control none -k regex:"k_block_gram|k_dgemm" --csv --log-file gpurun_out/small107.csv python tools/one_eval.py > /dev/null 2>&1; echo ncu=$?
python - <<'P'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/small107.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
t=defaultdict(list)
for r in rows[1:]:
    try: t[r[ki][:70]].append(float(r[vi].replace(',','')))
    except: pass
for k,v in t.items(): print(k, len(v), round(sum(v)/len(v)/1e3,2), 'us avg', round(sum(v)/3e3,1), 'us per eval')
P
B="timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
for v in 3 0 1 2 4 5 6 3; do FSA_GEMM_EXPAND=$v $B > gpurun_out/b107_$v.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/b107_$v.json').read().strip().splitlines()[-1]); t=d['timers_ms']; print('expand variant $v', round(d['ms_per_step'],3), d['clocks']['sm_mhz'], {k:t[k] for k in ('setup_trsm','setup_fitc','setup_sigma_m','probe_expand')})"; done
