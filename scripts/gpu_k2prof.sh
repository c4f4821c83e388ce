#!/bin/bash
O=gpurun_out/k2prof; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:'k2_alpha_beta' -s 4 -c 1 -o $O/k2_c2 python bench.py --config c2 --steps 2 --warmup 1 --eager --no-e2e --no-cpu-baseline > $O/ncu.log 2>&1
timeout -s KILL 120 python scripts/k2_steps.py > $O/k2_steps.txt 2>&1
echo done
