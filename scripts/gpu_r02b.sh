#!/bin/bash
# K8 / K9 bring-up: debug gradients, the joint tests, one joint_grad bench each for c3 / p124, launch list.
O=gpurun_out/r02b; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 python scripts/exp/jgrad_debug.py > $O/debug.log 2>&1; echo "debug exit $?" >> $O/debug.log
timeout -s KILL 900 python -m pytest tests/test_joint.py tests/test_canaries.py -q -p no:cacheprovider -x -s > $O/pytest_joint.log 2>&1; echo "exit $?" >> $O/pytest_joint.log
timeout -s KILL 600 python bench.py --mode joint_grad --no-cpu-baseline > $O/bench_joint_grad_c3.json 2> $O/bench_joint_grad_c3.err
timeout -s KILL 600 python bench.py --mode joint_grad --config p124 --no-cpu-baseline > $O/bench_joint_grad_p124.json 2> $O/bench_joint_grad_p124.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_jg_c3.csv python bench.py --mode joint_grad --steps 2 --warmup 3 --eager --no-cpu-baseline > $O/ncu.log 2>&1
echo done
