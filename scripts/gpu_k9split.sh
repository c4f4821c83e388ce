#!/bin/bash
O=gpurun_out/k9split; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for d in 4 5 6 7; do echo "dbg $d"; RNNT_K9_DEBUG=$d timeout -s KILL 300 python bench.py --mode joint_grad --steps 1 --warmup 1 --eager --no-cpu-baseline 2>&1 >/dev/null | grep "^K9" | tail -1; done > $O/summary.txt 2>&1
