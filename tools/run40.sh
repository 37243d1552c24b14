timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmm_v3 -s 2 -c 1 -o gpurun_out/ncu_spmm_v3 python tools/spmm_one.py > gpurun_out/ncu40.log 2>&1; echo ncu=$?
