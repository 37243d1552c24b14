# ncu --set full of one k_spmm_ms launch (config 2, k = 51; EPB=2, EPF=4)
export FSA_SPMM_EPB=2 FSA_SPMM_EPF=4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmm_ms -s 2 -c 1 -o gpurun_out/ncu_spmm_ms python tools/spmm_one.py > gpurun_out/ncu34.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu34.log
