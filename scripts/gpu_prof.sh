#!/bin/bash
# One gpurun call: remaining GPU tests, then the ncu launch list and one --set full capture of K1/K2/K3.
set -x
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_|k2_|k3_" -s 3 -c 3 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "done $?" >> gpurun_out/plain.log
