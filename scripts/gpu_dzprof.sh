#!/bin/bash
# per-role barrier waits of the dz kernel (RNNT_K6_DEBUG=4), c3 and p124 training steps
O=gpurun_out/dzp; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for c in p124 c3; do echo $c; RNNT_K6_DEBUG=4 timeout -s KILL 120 python bench.py --mode joint_grad --config $c --steps 1 --warmup 3 --eager --no-cpu-baseline --no-e2e 2>&1 | grep "K6 cycles" | tail -2; done > $O/roles.txt
