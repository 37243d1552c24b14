python -m pytest tests/test_gpu_ozaki.py tests/test_cpp_shim.py tests/test_fsagp_facade.py -x -q 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 3000 --launch-count 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/ncu_c4.log 2>&1; echo ncu_rc=$?
python tools/launch_summary.py gpurun_out/launches_c4.csv gpurun_out/launches_c4.txt "config 4" > /dev/null; head -16 gpurun_out/launches_c4.txt
ncu --set full --clock-control none -k regex:k_oz_gemm --launch-skip 20 -c 1 -o gpurun_out/ncu_c4_gemm python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/ncu_c4_gemm.log 2>&1; echo ncu2_rc=$?
