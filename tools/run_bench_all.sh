# round-2 measurement batch (results -> gpurun_out/, summaries copied to profiles/ by hand)
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; echo ref=$?
timeout 1200 python bench.py --config 3 --steps 3 --warmup 1 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
FSA_OZ_PAIR=0 timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/bench_c4_nopair.json 2> gpurun_out/bench_c4_nopair.err; echo c4np=$?
timeout 900 python bench.py --config 5 --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 --launch-count 1200 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?
python tools/launch_summary.py gpurun_out/launches_c2.csv gpurun_out/launches_c2.txt "round 2 config 2" > /dev/null
timeout 900 compute-sanitizer --tool memcheck --log-file gpurun_out/sanitizer_memcheck.txt python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san1.log 2>&1; echo memcheck=$?
timeout 900 compute-sanitizer --tool synccheck --log-file gpurun_out/sanitizer_synccheck.txt python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san2.log 2>&1; echo synccheck=$?
timeout 900 compute-sanitizer --tool racecheck --log-file gpurun_out/sanitizer_racecheck.txt python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san3.log 2>&1; echo racecheck=$?
tail -3 gpurun_out/sanitizer_*.txt
