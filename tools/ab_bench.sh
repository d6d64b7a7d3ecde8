#!/bin/bash
# A/B of an env knob on the N-GPU bench in one box: tools/ab_bench.sh N VAR [args...]
N=$1; VAR=$2; shift 2
for rep in 1 2; do
for v in 0 1; do
  env $VAR=$v timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + rep * 10 + v)) bench.py --gpus $N --steps 40 --warmup 5 --no-e2e "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', d['config']['workload'], round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step'],3), 'ms', {k: round(x,3) for k,x in d['kernel_ms_per_step'].items()})"
done; done
