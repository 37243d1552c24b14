# SpMM: 8 warps per CTA (two per row tile) vs 4
TAG=v3 python tools/spmm_ab.py
for mb in 3 4 5; do FSA_SPMM_W8=$mb TAG=v4-minb$mb python tools/spmm_ab.py; done
FSA_SPMM_W8=4 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -2
