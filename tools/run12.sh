python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest.log
B="timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0"
$B > gpurun_out/b_graph.json 2> gpurun_out/b_graph.err
FSA_NO_GRAPH=1 $B > gpurun_out/b_nograph.json 2> gpurun_out/b_nograph.err
python -m pytest tests/test_gpu_configs.py -q -s 2>&1 | grep -E "config|passed|failed"
