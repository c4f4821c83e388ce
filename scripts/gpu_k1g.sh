#!/bin/bash
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do
for gm in 8 16; do
  for dt in bf16 f16 f32; do
    RNNT_K1_GMAX=$gm timeout 300 python bench.py --dtype $dt --no-e2e --no-cpu-baseline --steps 50 > gpurun_out/k1g_${gm}_${dt}_$rep.json 2>/dev/null
  done
done
done
