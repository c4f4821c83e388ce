#!/bin/bash
O=gpurun_out/k9prof; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:'k9_dw' -s 1 -c 1 -o $O/k9_2sm python bench.py --mode joint_grad --config p124 --steps 1 --warmup 1 --eager --no-cpu-baseline > $O/ncu1.log 2>&1
RNNT_K9_CLUSTER=1 timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:'k9_dw' -s 1 -c 1 -o $O/k9_1 python bench.py --mode joint_grad --config p124 --steps 1 --warmup 1 --eager --no-cpu-baseline > $O/ncu2.log 2>&1
echo done
