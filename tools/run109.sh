# final round-2 batch: checked build suite, default suite, smoke, bench lines of all configs, launch list
FSA_LIB=$PWD/build/checked/libfsa_b200.so timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/checked_tests.txt 2>&1; tail -2 gpurun_out/checked_tests.txt
FSA_LIB=$PWD/build/checked/libfsa_b200.so timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee -a gpurun_out/checked_tests.txt
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/run105.sh
