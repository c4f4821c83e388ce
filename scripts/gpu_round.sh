#!/bin/bash
# Round check: all GPU tests, smoke(), the default bench line (with e2e and cpu_baseline) and the joint line.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout -s KILL 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "bench exit $?" >> gpurun_out/bench_c3.err
timeout -s KILL 600 python bench.py --mode joint > gpurun_out/bench_joint.json 2> gpurun_out/bench_joint.err
echo "bench exit $?" >> gpurun_out/bench_joint.err
