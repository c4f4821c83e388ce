#!/bin/bash
# K6<grad> diagnostics: per-role cycle split (RNNT_K6_DEBUG=4), then one ncu --set full capture of K6<grad>.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
RNNT_K6_DEBUG=4 timeout -s KILL 300 python bench.py --mode joint_grad --no-e2e --no-cpu-baseline --steps 2 --warmup 3 --eager > gpurun_out/k6g_dbg.json 2> gpurun_out/k6g_dbg.err
CMD="python bench.py --mode joint_grad --no-e2e --no-cpu-baseline --steps 1 --warmup 3 --eager"
timeout -s KILL 300 $CMD > gpurun_out/k6g_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k6_joint_lse<1" -c 1 \
    -o gpurun_out/k6grad_full $CMD > gpurun_out/k6g_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/k6g_ncu.log
