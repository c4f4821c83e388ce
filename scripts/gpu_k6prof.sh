#!/bin/bash
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for d in 4 5 6 7; do
  RNNT_K6_DEBUG=$d timeout -s KILL 300 python bench.py --mode joint --no-e2e --no-cpu-baseline --steps 3 --warmup 3 --eager > gpurun_out/k6prof_$d.json 2> gpurun_out/k6prof_$d.err
done
