#!/bin/bash
# Round evidence on one B200 (run via gpurun): smoke, GPU tests, bench line, launch list, ncu captures.
P=gpurun_out/ev
mkdir -p $P
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $P/smoke.log 2>&1; echo smoke=$?
timeout -s KILL 1500 python -m pytest tests -m gpu -q > $P/pytest.log 2>&1; echo pytest=$?
timeout -s KILL 900 python bench.py > $P/bench.json 2> $P/bench.err; echo bench=$?
A="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-optim"
timeout -s KILL 300 python bench.py $A > $P/plain.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/launches.csv python bench.py $A > $P/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:gemm2 -s 18 -c 6 -o $P/gemm_full python bench.py $A > $P/ncu_gemm.log 2>&1; echo ncu_gemm=$?
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:"gate_kernel|gate_dl|slot_|dispatch|combine|dwg|zero_" -s 33 -c 11 -o $P/other_full python bench.py $A > $P/ncu_other.log 2>&1; echo ncu_other=$?
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:update_kernel -s 1 -c 1 -o $P/optim_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $P/ncu_optim.log 2>&1; echo ncu_optim=$?
