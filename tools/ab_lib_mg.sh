#!/bin/bash
# Same-box A/B of two builds of libmoe.so on the N-GPU bench, interleaved:
#   tools/ab_lib_mg.sh N ab/libmoe_old.so [reps] [bench args...]
N=$1; OLD=$2; REPS=${3:-2}; shift 3
for rep in $(seq $REPS); do
for v in old new; do
  if [ $v = old ]; then LIBP=$(realpath $OLD); else LIBP=""; fi
  MOE_LIB_PATH=$LIBP timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29800 + rep * 10 + ${#v})) bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-optim "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'], round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step'],3), 'ms', {k: round(x,3) for k,x in d['kernel_ms_per_step'].items()}, round(d['a2a']['egress_GB/s'] or 0))"
done; done
