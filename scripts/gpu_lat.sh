#!/bin/bash
# Lattice-engine iteration: its GPU tests, bench line, and the ncu launch list of a short lattice run.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_lattice.py tests/test_canaries.py -q -x -p no:cacheprovider > gpurun_out/pytest_lat.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_lat.log
timeout 600 python bench.py --mode lattice --no-e2e --no-cpu-baseline > gpurun_out/bench_lat.json 2> gpurun_out/bench_lat.err
CMD="python bench.py --mode lattice --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_lat.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_lat.csv $CMD > gpurun_out/ncu_lat.log 2>&1
echo "ncu done $?" >> gpurun_out/plain_lat.log
