#!/bin/bash
# K6 forward per-role waits (RNNT_K6_DEBUG=4) with ablations: +1 no tanh, +16 no f/g loads, +2 no epilogue math
O=gpurun_out/k6r; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for c in p124 c3; do for d in 4 5 20 21 6 23; do echo "$c dbg=$d"; RNNT_K6_DEBUG=$d timeout -s KILL 120 python bench.py --mode joint --config $c --steps 1 --warmup 3 --eager --no-cpu-baseline --no-e2e 2>&1 | grep "K6 cycles" | tail -1; done; done > $O/roles.txt
