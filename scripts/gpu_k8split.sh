#!/bin/bash
# K8: per-chunk accumulator hand-over (default at H = 512) vs one hand-over (RNNT_K8_SPLIT=0)
out=gpurun_out/k8split.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 400 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/k8split_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/k8split_pytest.log)" >> $out
for rep in 1 2 3; do for v in 1 0; do for c in p124 c3; do
  RNNT_K8_SPLIT=$v timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('split=$v', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done; done
for v in 1 0; do for c in p124 c3; do
  echo "split=$v $c $(RNNT_K8_SPLIT=$v RNNT_K8_DEBUG=4 timeout -s KILL 120 python bench.py --mode joint_grad --config $c --steps 1 --warmup 3 --eager --no-cpu-baseline --no-e2e 2>&1 | grep 'K8 pair' | tail -1)" >> $out
done; done
O=gpurun_out/k8sl; mkdir -p $O
for v in 1 0; do for cfg in p124 c3; do
  RNNT_K8_SPLIT=$v timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/l_${v}_$cfg.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 3 --eager --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "split=$v $cfg $(python scripts/launch_summary.py $O/l_${v}_$cfg.csv | grep k8_)"; done; done >> $out 2>&1
