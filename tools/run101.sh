# where the e2e path's extra ~2 ms goes: geometry build timing + its kernel list
STAGE=1 timeout 300 python tools/e2e_parts.py 2>&1 | tail -2
STAGE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/geo101.csv python tools/e2e_parts.py > /dev/null 2>&1; echo ncu=$?
python - <<'P'
import csv,re
rows=list(csv.reader(open('gpurun_out/geo101.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
data=[(re.sub(r'\(.*','',r[ki])[-60:], float(r[vi].replace(',',''))/1e3) for r in rows[hi+1:] if len(r)>vi]
# last geometry build = last len/6 launches (6 builds, after kmeans etc.): print the last 1/6th
# find last occurrence of the first kernel of a build
names=[d[0] for d in data]
last=len(names)-1-names[::-1].index(names[-1])
# heuristic: print the final 60 launches
tot=0
for nme,t in data[-70:]:
    print(f"{t:8.1f} {nme}")
P
