#!/bin/bash
# Same-box A/B of two builds of libmoe.so on the 1-GPU bench, interleaved:
#   tools/ab_lib.sh ab/libmoe_old.so [reps] [bench args...]
# "new" is the in-tree paper_2305_13525_b200/libmoe.so.
OLD=$1; REPS=${2:-3}; shift 2
for rep in $(seq $REPS); do
for v in old new; do
  if [ $v = old ]; then LIBP=$OLD; else LIBP=""; fi
  MOE_LIB_PATH=$LIBP timeout -s KILL 300 python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['config']['workload'], round(d['value']/1e6,3), 'M tok/s', round(d['ms_per_step'],3), 'ms', {k: round(x,3) for k,x in d['kernel_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
done; done
