python -m pytest tests/test_cpp_shim.py -x -q > /dev/null 2>&1
./build/shim_example; echo shim_rc=$?
timeout 300 python tools/spmm_attr.py > gpurun_out/spmm_attr_ws.log 2>&1; head -4 gpurun_out/spmm_attr_ws.log
FSA_SPMM_KERNEL=rt timeout 300 python tools/spmm_attr.py > gpurun_out/spmm_attr_rt.log 2>&1; head -4 gpurun_out/spmm_attr_rt.log
