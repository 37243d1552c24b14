python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest.log
timeout 300 python tools/spmm_attr.py > gpurun_out/spmm_attr_ws.log 2>&1; head -3 gpurun_out/spmm_attr_ws.log
ncu --set full --import-source on --clock-control none -k regex:k_spmm_ws -c 1 -o gpurun_out/ncu_ws python tools/spmm_one.py > gpurun_out/ncu_ws.log 2>&1; echo ncu_ws=$?
FSA_SPMM_KERNEL=rt ncu --set full --import-source on --clock-control none -k regex:k_spmm_rt -c 1 -o gpurun_out/ncu_rt python tools/spmm_one.py > gpurun_out/ncu_rt.log 2>&1; echo ncu_rt=$?
