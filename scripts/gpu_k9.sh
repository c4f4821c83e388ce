#!/bin/bash
# K9 pair (cta_group::2) bring-up: gradients, joint tests, K9 launch times (pair vs single-CTA clusters).
O=gpurun_out/k9; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 python scripts/exp/jgrad_debug.py > $O/debug.log 2>&1; echo "debug exit $?" >> $O/debug.log
timeout -s KILL 600 python -m pytest tests/test_joint.py tests/test_canaries.py -q -p no:cacheprovider -x > $O/pytest_joint.log 2>&1; echo "exit $?" >> $O/pytest_joint.log
for cfg in c3 p124; do for v in "RNNT_K9_X=0" "RNNT_K9_CLUSTER=1"; do
  env $v timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k8_dh|k9_dw' -c 6 --csv --log-file $O/${cfg}_$v.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 2 --eager --no-cpu-baseline > /dev/null 2>&1
  echo "$cfg $v"; python scripts/launch_summary.py $O/${cfg}_$v.csv
done; done > $O/summary.txt 2>&1
echo done
