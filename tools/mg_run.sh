#!/bin/bash
# Multi-GPU evidence on N GPUs of one box (run via gpurun --gpus N): multi-process parity
# tests, then bench lines for the BASELINE configs that fit N GPUs (NVLink counters included).
N=${1:-2}
P=gpurun_out/mg$N
mkdir -p $P
nvidia-smi topo -m > $P/topo.txt 2>&1
timeout -s KILL 1200 python -m pytest tests/test_gpu_multi.py -q -rs > $P/pytest.log 2>&1; echo pytest=$?
timeout -s KILL 600 python -m pytest tests/test_gpu_emulated.py -q -x -m gpu -k "exchange_parity" > $P/emu.log 2>&1; echo emu=$?
run() {  # name, args...
  local name=$1; shift
  timeout -s KILL 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 30 --warmup 5 --no-optim --no-e2e "$@" \
    > $P/bench_$name.json 2> $P/bench_$name.err; echo bench_$name=$?
}
run 13b
run 27b --config 2.7b
run 67b_dtd --config 6.7b --gt 2
run 67b_nvls --config 6.7b --gt 2 --nvls
run 67b_van --config 6.7b --gt 2 --vanilla
if [ $N -ge 4 ]; then
  run 27b_tp2 --config 2.7b --gt 2
  run 27b_tp4 --config 2.7b --gt 4
  run 27b_tp4_nvls --config 2.7b --gt 4 --nvls
  run 27b_tp4_van --config 2.7b --gt 4 --vanilla
  run 67b_tp2ep2_nvls --config 6.7b --gt 2 --nvls
fi
