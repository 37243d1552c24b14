export FSA_LIB=$PWD/build/checked/libfsa_b200.so
echo "# round 2 end: the GPU test suite and smoke() on the bounds-checked, launch-synchronous build"
echo "# (make -C paper_2405_14492_b200/csrc checked; FSA_CHECKED: index checks in the gather / scatter"
echo "# kernels incl. k_spmm_v3's staged offsets and tile ranges + cudaDeviceSynchronize after every"
echo "# launch; compute-sanitizer is closed on this pool)"
echo "# FSA_LIB=build/checked/libfsa_b200.so"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
