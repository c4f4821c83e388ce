#!/bin/bash
# k9_reduce / k7_pred_sum with eight loads in flight: parity, launch lists, training-step lines
out=gpurun_out/reduce8.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 500 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/reduce8_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/reduce8_pytest.log)" >> $out
for cfg in p124 c3; do
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r8_$cfg.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 3 --eager --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "$cfg $(python scripts/launch_summary.py gpurun_out/r8_$cfg.csv | grep -E 'k9_reduce|k7_pred_sum' | tr '\n' ' ')" >> $out
done
for rep in 1 2; do for c in p124 c3; do
  timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done
