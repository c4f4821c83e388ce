#!/bin/bash
# K6<grad> as the two-operand-TMA dz kernel (default) vs k6_joint_lse<true> loading h (RNNT_K6_DZTMA=0)
mkdir -p gpurun_out; out=gpurun_out/dztma.txt; rm -f $out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py -q -x -m gpu -p no:cacheprovider > gpurun_out/dztma_pytest.log 2>&1
echo "pytest exit $?" >> $out
tail -2 gpurun_out/dztma_pytest.log >> $out
for rep in 1 2; do
  for dz in 1 0; do
    for c in p124 c3; do
      RNNT_K6_DZTMA=$dz timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('dztma=$dz', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
    done
  done
done
O=gpurun_out/dzl; mkdir -p $O
for cfg in p124 c3; do
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_${cfg}.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 3 --eager --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "$cfg"; python scripts/launch_summary.py $O/launches_${cfg}.csv; done > $O/summary.txt 2>&1
