#!/bin/bash
# per-role wait cycles of K8 (RNNT_K8_DEBUG=4) and K9 (RNNT_K9_DEBUG=4) in the training step, p124 and c3
O=gpurun_out/k89p; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for c in p124 c3; do echo $c; RNNT_K8_DEBUG=4 RNNT_K9_DEBUG=4 timeout -s KILL 120 python bench.py --mode joint_grad --config $c --steps 1 --warmup 3 --eager --no-cpu-baseline --no-e2e 2>&1 | grep -i "cycles" | tail -4; done > $O/roles.txt
