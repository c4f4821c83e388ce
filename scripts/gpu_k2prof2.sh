#!/bin/bash
O=gpurun_out/k2prof2; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 ncu --set full --import-source on --clock-control none -k regex:'k2_alpha_beta' -s 2 -c 1 -o $O/k2_u50 python scripts/exp/k2_long.py 50 > $O/ncu.log 2>&1
echo done
