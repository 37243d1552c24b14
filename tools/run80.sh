timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "probe or fitc" --timeout 300 -p no:cacheprovider 2>&1 | tail -3
