#!/bin/bash
O=gpurun_out/k1prof; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:'k1_lse' -s 4 -c 1 -o $O/k1_bf16 python bench.py --dtype bf16 --steps 2 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
echo done
