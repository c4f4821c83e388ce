#!/bin/bash
# K8 pair (cta_group::2) bring-up: gradients, joint tests, K8 / K9 launch times, pair vs the 2-D cluster kernel.
O=gpurun_out/k8; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 python scripts/exp/jgrad_debug.py > $O/debug.log 2>&1; echo "debug exit $?" >> $O/debug.log
timeout -s KILL 600 python -m pytest tests/test_joint.py tests/test_canaries.py -q -p no:cacheprovider -x > $O/pytest_joint.log 2>&1; echo "exit $?" >> $O/pytest_joint.log
for cfg in c3 p124; do for v in "RNNT_K8_X=0" "RNNT_K8_RT=4"; do
  env $v timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k8_dh|k9_dw' -c 6 --csv --log-file $O/${cfg}_$v.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 2 --eager --no-cpu-baseline > /dev/null 2>&1
  echo "$cfg $v"; python scripts/launch_summary.py $O/${cfg}_$v.csv
done; done > $O/summary.txt 2>&1
timeout -s KILL 600 python bench.py --mode joint_grad --no-cpu-baseline > $O/bench_joint_grad_c3.json 2> $O/bench_joint_grad_c3.err
timeout -s KILL 600 python bench.py --mode joint_grad --config p124 --no-cpu-baseline > $O/bench_joint_grad_p124.json 2> $O/bench_joint_grad_p124.err
echo done
