#!/bin/bash
# ncu --set full of K1 and K3 at p124 fp16 (V = 500: 64-bit row-group kernels), one bench step (eager launch)
O=gpurun_out/p124h; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:'k1_lse|k3_grad' -s 8 -c 8 -o $O/p124h python bench.py --config p124 --dtype f16 --steps 1 --warmup 2 --eager --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
echo "exit $?" >> $O/ncu.log
