#!/bin/bash
# Same-box weak-scaling curve of the default workload (1.3B layer, 16k tokens per GPU,
# experts over N GPUs): N = 1, 2, 4 back to back on one 4-GPU box (run via gpurun --gpus 4).
P=gpurun_out/scale
mkdir -p $P
for N in 1 2 4; do
  if [ $N = 1 ]; then
    timeout -s KILL 400 python bench.py --no-cpu-baseline --no-optim > $P/n$N.json 2> $P/n$N.err; echo n$N=$?
  else
    timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + N)) bench.py --gpus $N --no-optim > $P/n$N.json 2> $P/n$N.err; echo n$N=$?
  fi
done
