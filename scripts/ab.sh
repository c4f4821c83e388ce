#!/bin/bash
# A/B: bench the in-tree library and paper_2303_10384_b200/lib/ab/*.so alternately on one box.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do
  for lib in paper_2303_10384_b200/lib/librnnt_b200.so paper_2303_10384_b200/lib/ab/*.so; do
    n=$(basename $lib .so)
    RNNT_B200_LIB=$PWD/$lib python bench.py --no-e2e --no-cpu-baseline ${AB_ARGS} > gpurun_out/ab_${n}_$rep.json 2>/dev/null
  done
done
