#!/bin/bash
O=gpurun_out/k8split; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for cfg in c3 p124; do echo "$cfg"; RNNT_K8_DEBUG=4 timeout -s KILL 300 python bench.py --mode joint_grad --config $cfg --steps 1 --warmup 1 --eager --no-cpu-baseline 2>&1 >/dev/null | grep "^K8" | tail -1; done > $O/summary.txt 2>&1
