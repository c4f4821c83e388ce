#!/bin/bash
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py -q -x -p no:cacheprovider --timeout 200 > gpurun_out/pytest_joint.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_joint.log
grep -q "pytest exit 0" gpurun_out/pytest_joint.log || exit 0
for d in ${DBG:-0 1 2 3}; do
  RNNT_K6_DEBUG=$d timeout -s KILL 300 python bench.py --mode joint --no-e2e --no-cpu-baseline --steps 30 --warmup 3 > gpurun_out/k6exp_$d.json 2>&1
done
RNNT_K6_DEBUG=4 timeout -s KILL 300 python bench.py --mode joint --no-e2e --no-cpu-baseline --steps 3 --warmup 3 --eager > gpurun_out/k6prof_4.json 2> gpurun_out/k6prof_4.err
