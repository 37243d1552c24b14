# which GPU test stalls with the new SpMM kernels?
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_sharded.py -v -x --timeout 120 -p no:cacheprovider 2>&1 | grep -v "^$" | tail -40
