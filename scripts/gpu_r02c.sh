#!/bin/bash
# K8 2-D cluster version: debug gradients, joint tests, benches, launch list, ncu --set full of K8 and K9.
O=gpurun_out/r02c; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 python scripts/exp/jgrad_debug.py > $O/debug.log 2>&1; echo "debug exit $?" >> $O/debug.log
timeout -s KILL 900 python -m pytest tests/test_joint.py tests/test_canaries.py -q -p no:cacheprovider -x > $O/pytest_joint.log 2>&1; echo "exit $?" >> $O/pytest_joint.log
timeout -s KILL 600 python bench.py --mode joint_grad --no-cpu-baseline > $O/bench_joint_grad_c3.json 2> $O/bench_joint_grad_c3.err
timeout -s KILL 600 python bench.py --mode joint_grad --config p124 --no-cpu-baseline > $O/bench_joint_grad_p124.json 2> $O/bench_joint_grad_p124.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_jg_c3.csv python bench.py --mode joint_grad --steps 2 --warmup 3 --eager --no-cpu-baseline > $O/ncu.log 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:'k8_dh|k9_dw' -s 2 -c 2 -o $O/k89_full python bench.py --mode joint_grad --steps 1 --warmup 3 --eager --no-cpu-baseline > $O/ncu_full.log 2>&1
echo done
