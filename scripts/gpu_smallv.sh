#!/bin/bash
# K6 forward at small V with per-CTA MMAs (default now) -- parity and the p124 lines
out=gpurun_out/smallv.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 500 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/smallv_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/smallv_pytest.log)" >> $out
for rep in 1 2; do for c in "--mode joint --config p124" "--mode joint_grad --config p124" "--mode joint --config c3"; do
  timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done
