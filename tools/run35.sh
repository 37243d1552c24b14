# SpMM: union order A/B on the new kernel, and the ncu capture of the default variant
TAG=mask FLAGS=0,2,3,15 python tools/spmm_ab.py
FSA_UNION_ORDER=plain TAG=plain FLAGS=0,2,3,15 python tools/spmm_ab.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmm_ms -s 2 -c 1 -o gpurun_out/ncu_spmm_ms2 python tools/spmm_one.py > gpurun_out/ncu35.log 2>&1; echo ncu=$?
