# SpMM A/B: piece size 8 vs 16, ring depth, epilogue prefetch lead
TAG=p16n2f4 FLAGS=0 python tools/spmm_ab.py
for ns in 2 3 4; do for epf in 4 8; do FSA_SPMM_P=8 FSA_SPMM_NS=$ns FSA_SPMM_EPF=$epf TAG=p8n${ns}f${epf} FLAGS=0 python tools/spmm_ab.py; done; done
FSA_SPMM_NS=3 TAG=p16n3f4 FLAGS=0 python tools/spmm_ab.py
