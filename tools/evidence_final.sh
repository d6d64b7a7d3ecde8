#!/bin/bash
# Final evidence on one B200 (run via gpurun): the bench line first (cool box), then the
# ncu launch list of the same command and ncu --set full captures of the GEMMs and of the
# non-GEMM kernels of one step.
P=gpurun_out/evf
mkdir -p $P
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit,temperature.gpu --format=csv > $P/smi.txt 2>&1
timeout -s KILL 600 python bench.py > $P/bench.json 2> $P/bench.err; echo bench=$?
A="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-optim"
timeout -s KILL 400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $P/launches.csv python bench.py $A > $P/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
  -k regex:"gate_tc|slot_final|dispatch|combine_bwd_gate|dwg_tc" -s 10 -c 5 -o $P/small_full python bench.py $A \
  > $P/ncu_small.log 2>&1; echo ncu_small=$?
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 12 -c 6 \
  -o $P/gemm_full python bench.py $A > $P/ncu_gemm.log 2>&1; echo ncu_gemm=$?
