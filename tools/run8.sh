timeout 300 python tools/spmm_attr.py > gpurun_out/spmm_attr_ws.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest.log
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
$B > gpurun_out/b_ws_graph.json 2> gpurun_out/b_ws_graph.err
FSA_NO_GRAPH=1 $B > gpurun_out/b_ws_nograph.json 2> gpurun_out/b_ws_nograph.err
FSA_SPMM_KERNEL=rt $B > gpurun_out/b_rt_graph.json 2> gpurun_out/b_rt_graph.err
cat gpurun_out/spmm_attr_ws.log
