# union order A/B: mask order vs mask order with k-steps interleaved across pieces
FSA_UNION_ORDER=mask TAG=mask FLAGS=0 python tools/spmm_ab.py
TAG=interleave FLAGS=0 python tools/spmm_ab.py
FSA_SPMM_NS=3 TAG=interl-ns3 FLAGS=0 python tools/spmm_ab.py
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 2>&1 | tail -2
