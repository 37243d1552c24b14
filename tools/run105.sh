# round-2 session-4 measurement batch (results -> gpurun_out/, summaries copied to profiles/r02c_* by hand)
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; echo ref=$?
timeout 1200 python bench.py --config 3 --steps 3 --warmup 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 900 python bench.py --config 5 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
timeout 900 ncu --nvtx --nvtx-include "one_eval/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/one_eval.py > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?
python tools/launch_summary.py gpurun_out/launches_c2.csv gpurun_out/launches_c2.txt "round 2 session 4 (end), config 2: three loglik+grad evaluations" > /dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_gemm|k_oz_expand|k_spmm_v3|k_xr_dot_max|k_oz_planes_y" --launch-skip 300 --launch-count 5 -o gpurun_out/sweep_full python tools/one_eval.py > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
timeout 300 python tools/one_eval.py 2>&1 | tail -3
for f in bench_c2 ref_c2 bench_c3 bench_c4 bench_c5; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d.get('ms_per_step'), d.get('value'), (d.get('e2e') or {}).get('value'), d.get('clocks'))"; done
