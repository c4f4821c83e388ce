#!/bin/bash
# One gpurun call per iteration: GPU tests, full bench line, then (only if those exit 0) the ncu launch
# list and one --set full capture of K1/K2/K3 on the same short command.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
[ -n "$NO_NCU" ] && exit 0
grep -q "pytest exit 0" gpurun_out/pytest_gpu.log || exit 0
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${NCU_BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_|k2_|k3_" -s 3 -c 3 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu done $?" >> gpurun_out/plain.log
