#!/bin/bash
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py -q -x -p no:cacheprovider --timeout 120 > gpurun_out/pytest_joint.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_joint.log
grep -q "pytest exit 0" gpurun_out/pytest_joint.log || exit 0
for rep in 1 2; do for cl in 2 1; do
  RNNT_K6_CLUSTER=$cl timeout -s KILL 300 python bench.py --mode joint --no-e2e --no-cpu-baseline --steps 30 --warmup 3 > gpurun_out/k6cl_${cl}_$rep.json 2>/dev/null
  RNNT_K6_CLUSTER=$cl timeout -s KILL 300 python bench.py --mode joint --config p124 --no-e2e --no-cpu-baseline --steps 30 --warmup 3 > gpurun_out/k6cl_p124_${cl}_$rep.json 2>/dev/null
done; done
