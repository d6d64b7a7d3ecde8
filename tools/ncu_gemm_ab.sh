#!/bin/bash
# ncu cycles of the six expert GEMMs of one step for two builds (MOE_LIB_PATH A/B)
OLD=$1
A="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-optim"
for v in old new; do
  if [ $v = old ]; then export MOE_LIB_PATH=$(realpath $OLD); else unset MOE_LIB_PATH; fi
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm2 -s 18 -c 6 --csv python bench.py $A > gpurun_out/ncu_ab_$v.csv 2>/dev/null
done
