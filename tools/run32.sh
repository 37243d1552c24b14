# SpMM A/B: batched epilogue loads (FSA_SPMM_EPB) and late L2 prefetch of the epilogue rows (FSA_SPMM_EPF)
FSA_SPMM=rt TAG=rt python tools/spmm_ab.py
for epb in 1 2; do for epf in 0 2 4 8; do FSA_SPMM_EPB=$epb FSA_SPMM_EPF=$epf TAG=b${epb}f${epf} FLAGS=0 python tools/spmm_ab.py; done; done
FSA_SPMM_EPB=1 TAG=b1-attr FLAGS=2,3,15 python tools/spmm_ab.py
