FSA_SPMM_KERNEL=rt timeout 300 python tools/spmm_attr.py > gpurun_out/spmm_attr_rt.log 2>&1; head -4 gpurun_out/spmm_attr_rt.log
python -m pytest tests -m gpu -q --deselect tests/test_gpu_configs.py::test_config_nll_grad_matches_oracle[5] --deselect tests/test_gpu_configs.py::test_config5_bench_precond_matches_oracle > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest.log
