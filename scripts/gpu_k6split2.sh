#!/bin/bash
O=gpurun_out/k6split2; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for cfg in c3 p124; do for m in joint joint_grad; do echo "$cfg $m"; RNNT_K6_DEBUG=4 timeout -s KILL 120 python bench.py --mode $m --config $cfg --steps 1 --warmup 1 --eager --no-cpu-baseline 2>&1 >/dev/null | grep "^K6" | tail -2; done; done > $O/summary.txt 2>&1
