# session-4 profile of the current code: launch list of one_eval evaluations + full captures of the sweep kernels
timeout 900 ncu --nvtx --nvtx-include "one_eval/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/one_eval.py > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?
python tools/launch_summary.py gpurun_out/launches_c2.csv gpurun_out/launches_c2.txt "round 2 session 4, config 2: three loglik+grad evaluations" > /dev/null
head -30 gpurun_out/launches_c2.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_oz_gemm|k_oz_expand|k_spmm_v3|k_xr_dot_max|k_oz_planes_y" --launch-skip 300 --launch-count 5 -o gpurun_out/sweep_full python tools/one_eval.py > gpurun_out/ncu_full.log 2>&1; echo ncufull=$?
ls -la gpurun_out/
