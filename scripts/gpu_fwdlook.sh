#!/bin/bash
# K6 forward: rows' cell / lengths / label one tile ahead (default) vs in place (RNNT_K6_DEBUG=64)
out=gpurun_out/fwdlook.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 400 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/fwdlook_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/fwdlook_pytest.log)" >> $out
for rep in 1 2 3; do for v in 0 64; do for c in "--mode joint --config c3" "--mode joint --config p124" "--mode joint_grad --config c3" "--mode joint_grad --config p124"; do
  RNNT_K6_DEBUG=$v timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('dbg=$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
