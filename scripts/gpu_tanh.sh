#!/bin/bash
O=gpurun_out/tanh; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for d in 0 8 0 8; do RNNT_K6_DEBUG=$d timeout -s KILL 400 python scripts/exp/tanh_ab.py >> $O/summary.txt 2>> $O/err.txt; done
