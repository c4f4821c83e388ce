#!/bin/bash
# ncu --set full of one kernel (regex $KREGEX) on a short bench command ($BENCH_ARGS), after the same
# command exits 0 without ncu.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
$CMD > gpurun_out/plain_one.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-2} -c ${COUNT:-1} -o gpurun_out/${OUT:-one} $CMD > gpurun_out/ncu_one.log 2>&1
echo "ncu done $?" >> gpurun_out/plain_one.log
