python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo pytest_rc=$?; grep -E "passed|failed|FAILED" gpurun_out/pytest.log | tail -5
python -m pytest tests/test_gpu_configs.py -q -s 2>&1 | grep -E "^config|FITC|passed|failed" > gpurun_out/cfgtests.log; cat gpurun_out/cfgtests.log
