# expansion: direct-write 4-stage epilogue vs the staged 3-stage one
FSA_OZ_STAGED=1 WHICH=2 TAG=staged python tools/spmm_ab.py
WHICH=2 TAG=direct python tools/spmm_ab.py
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider 2>&1 | tail -2
