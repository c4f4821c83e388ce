#!/bin/bash
# K6 pair MMAs: joint tests, launch lists (pair vs multicast), joint / joint_grad benches.
O=gpurun_out/k6pair; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 120 python scripts/exp/jgrad_debug.py > $O/debug.log 2>&1; echo "debug exit $?" >> $O/debug.log
timeout -s KILL 240 python -m pytest tests/test_joint.py tests/test_canaries.py -q -p no:cacheprovider -x --timeout 60 > $O/pytest_joint.log 2>&1; echo "exit $?" >> $O/pytest_joint.log
for cfg in c3 p124; do for v in "RNNT_K6_PAIR=1" "RNNT_K6_PAIR=0"; do
  env $v timeout -s KILL 150 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k6_joint' -c 4 --csv --log-file $O/${cfg}_$v.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 1 --eager --no-cpu-baseline > /dev/null 2>&1
  echo "$cfg $v"; python scripts/launch_summary.py $O/${cfg}_$v.csv
done; done > $O/summary.txt 2>&1
for m in joint joint_grad; do for cfg in c3 p124; do
timeout -s KILL 150 python bench.py --mode $m --config $cfg --no-cpu-baseline > $O/bench_${m}_$cfg.json 2> $O/bench_${m}_$cfg.err; done; done
echo done
