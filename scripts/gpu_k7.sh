#!/bin/bash
O=gpurun_out/k7; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py tests/test_canaries.py -q -p no:cacheprovider -x --timeout 60 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for cfg in c3 p124; do for v in "RNNT_K7_UNITS=0" "RNNT_K7_UNITS=1"; do
  env $v timeout -s KILL 150 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k7_' -c 4 --csv --log-file $O/${cfg}_$v.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 1 --eager --no-cpu-baseline > /dev/null 2>&1
  echo "$cfg $v"; python scripts/launch_summary.py $O/${cfg}_$v.csv
done; done > $O/summary.txt 2>&1
