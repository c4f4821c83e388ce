#!/bin/bash
# ncu launch lists of the joint training step with and without K6<grad> reusing the forward's h
O=gpurun_out/hrl; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for hr in 1 0; do for cfg in p124 c3; do
RNNT_K6_HREUSE=$hr timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_${cfg}_hr$hr.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 3 --eager --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "$cfg hreuse=$hr"; python scripts/launch_summary.py $O/launches_${cfg}_hr$hr.csv; done; done > $O/summary.txt 2>&1
for hr in 1 0; do RNNT_K6_HREUSE=$hr RNNT_K6_DEBUG=4 timeout -s KILL 120 python bench.py --mode joint_grad --config p124 --steps 1 --warmup 3 --eager --no-cpu-baseline --no-e2e 2>&1 | grep "K6 cycles" | tail -2; done > $O/roles.txt
