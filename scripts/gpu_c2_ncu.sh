#!/bin/bash
# ncu --set full of K1 / K3 at c2 (four utterance chunks), one bench step (eager)
O=gpurun_out/c2n; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 900 ncu --set full --clock-control none -k regex:'k1_lse|k3_grad' -s 16 -c 8 -o $O/c2 python bench.py --config c2 --steps 1 --warmup 3 --eager --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
echo "exit $?" >> $O/ncu.log
