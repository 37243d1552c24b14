# the NCCL / torchrun code path at one rank (strong mode = the row-sharded context), config 2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --mode strong --no-cpu-baseline --no-dmma-arm --e2e-steps 1 > gpurun_out/b75.json 2> gpurun_out/b75.err; echo rc=$?
python -c "
import json;d=json.loads(open('gpurun_out/b75.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['value'], d['nll'], d['config']['parallelism'], d.get('scaling'))"
tail -3 gpurun_out/b75.err
