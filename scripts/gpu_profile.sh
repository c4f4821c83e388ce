#!/bin/bash
# Launch list + one ncu --set full capture of K1/K2/K3 on the bench command (each after a clean plain run).
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${PROF_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_|k2_|k3_" -s 12 -c 12 -o gpurun_out/prof $CMD > gpurun_out/ncu_full.log 2>&1
echo "done $?" >> gpurun_out/plain.log
