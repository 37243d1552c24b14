# measurement after the base-256 digit format: config 2 full line, launch list, ncu of the Ozaki kernels
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
timeout 900 ncu --nvtx --nvtx-include "one_eval/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/one_eval.py > gpurun_out/ncu_l.log 2>&1; echo ncu=$?
python tools/launch_summary.py gpurun_out/launches_c2.csv gpurun_out/launches_c2.txt "round 2 end config 2: three loglik+grad evaluations (base-256 Ozaki digits)" > /dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_oz_expand -s 2 -c 1 -o gpurun_out/ncu_expand_b256 python tools/spmm_one.py 2 > gpurun_out/ncu_x.log 2>&1; echo ncux=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_oz_gemm -s 2 -c 1 -o gpurun_out/ncu_gemm_b256 python tools/spmm_one.py 1 > gpurun_out/ncu_g.log 2>&1; echo ncug=$?
