#!/bin/bash
# A/B: alternate two library builds, 2 runs each
L=paper_2405_14492_b200/libfsa_b200.so
for r in 1 2; do
for v in $@; do
  cp abl/lib_$v.so $L
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_${v}_$r.json 2>/dev/null
done
done
