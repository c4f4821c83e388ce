#!/bin/bash
O=gpurun_out/jgl; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for cfg in c3 p124; do
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_$cfg.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 3 --eager --no-cpu-baseline > /dev/null 2>&1
echo $cfg; python scripts/launch_summary.py $O/launches_$cfg.csv; done > $O/summary.txt 2>&1
