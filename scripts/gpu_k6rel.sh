#!/bin/bash
O=gpurun_out/k6rel; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py tests/test_canaries.py -q -p no:cacheprovider -x --timeout 60 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for cfg in c3 p124; do
  timeout -s KILL 150 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k6_joint' -c 4 --csv --log-file $O/${cfg}.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 1 --eager --no-cpu-baseline > /dev/null 2>&1
  echo "$cfg"; python scripts/launch_summary.py $O/${cfg}.csv
  for m in joint joint_grad; do timeout -s KILL 120 python bench.py --mode $m --config $cfg --steps 60 --no-cpu-baseline > $O/b.json 2>/dev/null; python -c "import json; d=json.load(open('$O/b.json')); print('$cfg $m', round(d['ms_per_step'],3), round(d['value']), d['clocks']['sm_mhz'])"; done
done > $O/summary.txt 2>&1
