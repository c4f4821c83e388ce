#!/bin/bash
# fair re-run of the k6_dz_2sm TMA-store A/B (RNNT_K6_DEBUG=32 no longer touches the forward builders)
out=gpurun_out/dzstore2.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 400 python -m pytest tests/test_joint.py -q -x -m gpu -p no:cacheprovider -k "ab_paths or loss_grad_matches" > gpurun_out/dzstore2_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/dzstore2_pytest.log)" >> $out
for rep in 1 2 3; do for v in 0 32; do for c in p124 c3; do
  RNNT_K6_DEBUG=$v timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('dbg=$v', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done; done
