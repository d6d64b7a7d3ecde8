for kb in 200 144 96; do
for c in 1.3b 2.7b 6.7b; do
MOE_DX_BUDGET_KB=$kb timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-optim 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$kb', d['config']['workload'], round(d['value']/1e6,3), round(d['kernel_ms_per_step']['gate_bwd'],3))"
done; done
