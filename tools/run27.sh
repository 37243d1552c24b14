ncu --set full --import-source on --clock-control none -k regex:k_oz_expand -c 1 -o gpurun_out/ncu_expand python tools/spmm_one.py 2 > gpurun_out/ncu_expand.log 2>&1; echo e=$?
ncu --set full --import-source on --clock-control none -k regex:k_oz_gemm -c 1 -o gpurun_out/ncu_gemm python tools/spmm_one.py 1 > gpurun_out/ncu_gemm.log 2>&1; echo g=$?
