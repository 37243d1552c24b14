for mb in 5 6 7 8; do FSA_SPMM_MINB=$mb TAG=minb$mb python tools/spmm_ab.py; done
