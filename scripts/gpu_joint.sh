#!/bin/bash
# Fused-joint iteration: its GPU tests (own timeout: a barrier bug must not hang the box), then bench.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_joint.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_joint.log
grep -q "pytest exit 0" gpurun_out/pytest_joint.log || exit 0
timeout -s KILL 300 python bench.py --mode joint --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_joint.json 2> gpurun_out/bench_joint.err
echo "bench exit $?" >> gpurun_out/bench_joint.err
