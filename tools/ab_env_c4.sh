#!/bin/bash
# A/B of an environment switch on BASELINE config 4: ab_env_c4.sh VAR
for r in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export $1=1; else unset $1; fi
  timeout 600 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/abc4_${v}_$r.json 2>/dev/null
done
done
