python -m pytest tests/test_cpp_shim.py -x -q > /dev/null 2>&1
FSA_DEBUG=1 ./build/shim_example; echo shim_rc=$?
FSA_NO_GRAPH=1 ./build/shim_example; echo shim_nograph_rc=$?
