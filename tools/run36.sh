# SpMM A/B: lean v3 main loop vs k_spmm_ms; correctness of v3
FSA_SPMM=ms TAG=ms FLAGS=0 python tools/spmm_ab.py
for ns in 2 3; do for epb in 1 2; do FSA_SPMM_NS=$ns FSA_SPMM_EPB=$epb TAG=v3n${ns}b${epb} FLAGS=0 python tools/spmm_ab.py; done; done
TAG=v3-attr FLAGS=2 python tools/spmm_ab.py
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_sharded.py -x -q --durations=5 2>&1 | tail -9
