timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_oz_expand -s 2 -c 1 -o gpurun_out/ncu_expand python tools/spmm_one.py 2 > gpurun_out/ncu45.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_oz_gemm -s 2 -c 1 -o gpurun_out/ncu_gemm python tools/spmm_one.py 1 > gpurun_out/ncu45b.log 2>&1; echo ncu=$?
