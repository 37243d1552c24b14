#!/bin/bash
# A/B of an environment switch: ab_env.sh VAR  (runs VAR unset / VAR=1, twice each)
for r in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export $1=1; else unset $1; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abe_${v}_$r.json 2>/dev/null
done
done
