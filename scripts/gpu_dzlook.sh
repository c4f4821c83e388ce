#!/bin/bash
# k6_dz_2sm: rows' scalars one tile ahead (default) vs in place (RNNT_K6_DEBUG=64); parity, A/B, roles, launch lists
out=gpurun_out/dzlook.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 400 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/dzlook_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/dzlook_pytest.log)" >> $out
for rep in 1 2 3; do for v in 0 64; do for c in p124 c3; do
  RNNT_K6_DEBUG=$v timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('dbg=$v', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done; done
for v in 4 68; do for c in p124 c3; do
  echo "dbg=$v $c $(RNNT_K6_DEBUG=$v timeout -s KILL 120 python bench.py --mode joint_grad --config $c --steps 1 --warmup 3 --eager --no-cpu-baseline --no-e2e 2>&1 | grep 'K6 cycles' | tail -1)" >> $out
done; done
O=gpurun_out/dzll; mkdir -p $O
for v in 0 64; do for cfg in p124 c3; do
  RNNT_K6_DEBUG=$v timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/l_${v}_$cfg.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 3 --eager --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "dbg=$v $cfg $(python scripts/launch_summary.py $O/l_${v}_$cfg.csv | grep k6_dz)"; done; done >> $out 2>&1
