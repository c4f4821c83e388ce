#!/bin/bash
# Joint training-step iteration: the joint tests, then the c3 and p124 joint_grad benches.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py -q -x -p no:cacheprovider > gpurun_out/pytest_joint.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_joint.log
grep -q "pytest exit 0" gpurun_out/pytest_joint.log || exit 0
timeout -s KILL 300 python bench.py --mode joint_grad --no-e2e --no-cpu-baseline > gpurun_out/bench_jgrad.json 2>&1
timeout -s KILL 300 python bench.py --mode joint_grad --config p124 --no-e2e --no-cpu-baseline > gpurun_out/bench_jgrad_p124.json 2>&1
timeout -s KILL 300 python bench.py --mode joint_grad --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_jgrad.csv \
    python bench.py --mode joint_grad --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
