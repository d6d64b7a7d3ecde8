for cfg in 1.3b 2.7b 6.7b; do
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 30 --warmup 5 --config $cfg --no-optim > gpurun_out/m4_$cfg.json 2>gpurun_out/m4_$cfg.err
done
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 30 --warmup 5 --config 6.7b --vanilla --no-optim --no-e2e > gpurun_out/m4_6.7bvan.json 2>gpurun_out/m4_6.7bvan.err
