# round 2 re-entry: baseline check of the restored tree
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 3 --no-dmma-arm > gpurun_out/b30.json 2> gpurun_out/b30.err; echo bench=$?
tail -c 3000 gpurun_out/b30.json
