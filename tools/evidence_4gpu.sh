#!/bin/bash
# Multi-GPU evidence on one 4-GPU box (run via gpurun --gpus 4): parity tests + bench sweep.
P=gpurun_out/ev4
mkdir -p $P
timeout -s KILL 1500 python -m pytest tests/test_gpu_multi.py -q > $P/pytest_multi.log 2>&1; echo pytest=$?
run() {  # name N args...
  local name=$1 n=$2; shift 2
  timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29900 + RANDOM % 90)) bench.py --gpus $n "$@" > $P/$name.json 2> $P/$name.err; echo $name=$?
}
run 13b_n2 2
run 13b_n4 4
run 27b_n4_gt1 4 --config 2.7b --steps 30 --warmup 5 --no-e2e --no-optim
run 27b_n4_gt2 4 --config 2.7b --gt 2 --steps 30 --warmup 5 --no-e2e --no-optim
run 27b_n4_gt4 4 --config 2.7b --gt 4 --steps 30 --warmup 5 --no-e2e --no-optim
run 27b_n4_gt2_van 4 --config 2.7b --gt 2 --vanilla --steps 30 --warmup 5 --no-e2e --no-optim
run 27b_n2_gt1 2 --config 2.7b --steps 30 --warmup 5 --no-e2e --no-optim
run 27b_n2_gt2 2 --config 2.7b --gt 2 --steps 30 --warmup 5 --no-e2e --no-optim
run 67b_n4_dtd 4 --config 6.7b --steps 30 --warmup 5 --no-e2e --no-optim
run 67b_n4_van 4 --config 6.7b --vanilla --steps 30 --warmup 5 --no-e2e --no-optim
run 67b_n2_dtd 2 --config 6.7b --steps 30 --warmup 5 --no-e2e --no-optim
run 67b_n2_van 2 --config 6.7b --vanilla --steps 30 --warmup 5 --no-e2e --no-optim
