# SpMM A/B: bulk-copy gathers (FSA_SPMM_BULK) x ring depth x epilogue batching, L2 prefetch 4 pieces ahead
for bulk in 0 1; do for ns in 2 3; do for epb in 1 2; do
FSA_SPMM_BULK=$bulk FSA_SPMM_NS=$ns FSA_SPMM_EPB=$epb FSA_SPMM_EPF=4 TAG=u${bulk}n${ns}b${epb} FLAGS=0 python tools/spmm_ab.py
done; done; done
FSA_SPMM_BULK=1 FSA_SPMM_EPB=2 FSA_SPMM_EPF=4 TAG=bulk-attr FLAGS=2,3,15 python tools/spmm_ab.py
FSA_SPMM_BULK=1 FSA_SPMM_EPF=4 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --durations=5 2>&1 | tail -9
