#!/bin/bash
O=gpurun_out/k9abl; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for v in "RNNT_K9_DEBUG=0" "RNNT_K9_DEBUG=1" "RNNT_K9_DEBUG=2" "RNNT_K9_DEBUG=3"; do
  env $v timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k9_dw' -c 3 --csv --log-file $O/$v.csv python bench.py --mode joint_grad --steps 2 --warmup 2 --eager --no-cpu-baseline > /dev/null 2>&1
  echo "$v"; python scripts/launch_summary.py $O/$v.csv
done > $O/summary.txt 2>&1
