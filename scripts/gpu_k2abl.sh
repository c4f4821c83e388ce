#!/bin/bash
# K2 per-step cost with stores / operand loads ablated (build-time RNNT_K2_ABL variants; timing only)
out=gpurun_out/k2abl.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for v in base k2abl1 k2abl4 k2abl5; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  echo "== $v" >> $out
  RNNT_B200_LIB=$L timeout -s KILL 300 python scripts/k2_steps.py rnnt >> $out 2>&1
done
