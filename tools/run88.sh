# PDL launch_dependents trigger: parity + A/B timing against a -DFSA_NO_PDL_TRIGGER build
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do
  timeout 300 python tools/one_eval.py 2>&1 | tail -1 | sed 's/^/trig   /'
  FSA_LIB=$PWD/build/notrig/libfsa_b200.so timeout 300 python tools/one_eval.py 2>&1 | tail -1 | sed 's/^/notrig /'
done
for r in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export FSA_LIB=$PWD/build/notrig/libfsa_b200.so; else unset FSA_LIB; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-dmma-arm --e2e-steps 0 > gpurun_out/ab88_${v}_$r.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ab88_${v}_$r.json').read().strip().splitlines()[-1]); print('notrig=$v', round(d['ms_per_step'],3), round(d['pcg_ms'],3), repr(d['nll']), d['clocks']['sm_mhz'])"
done; done
