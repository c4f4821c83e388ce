#!/bin/bash
# A/B: K6<grad> loading the forward's h (default) vs recomputing it (RNNT_K6_HREUSE=0); joint parity first
mkdir -p gpurun_out; out=gpurun_out/hreuse.txt; rm -f $out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py -q -x -m gpu -p no:cacheprovider > gpurun_out/hreuse_pytest.log 2>&1
echo "pytest exit $?" >> $out
tail -2 gpurun_out/hreuse_pytest.log >> $out
for rep in 1 2; do
  for hr in 1 0; do
    for c in p124 c3; do
      RNNT_K6_HREUSE=$hr timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('hreuse=$hr', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
    done
  done
done
