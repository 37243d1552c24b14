# projection-chain L2 hints only (final form) + geometry readback folded: full GPU suite, smoke, bench
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm > gpurun_out/b104_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/b104_$r.json').read().strip().splitlines()[-1]); t=d['timers_ms']; print(round(d['ms_per_step'],3), round(d['e2e']['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['clocks']['sm_mhz'], {k:t[k] for k in ('cg_blas1','spmm','lowrank_project','lowrank_expand')})"; done
