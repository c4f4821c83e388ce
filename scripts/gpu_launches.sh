#!/bin/bash
# ncu launch list (per-launch durations) of a short bench command, after it exits 0 without ncu.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${PROF_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches${TAG}.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "done $?" >> gpurun_out/plain.log
