TAG=minb8 python tools/spmm_ab.py
FSA_SPMM_MINB7=1 TAG=minb7 python tools/spmm_ab.py
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/one_eval.py
