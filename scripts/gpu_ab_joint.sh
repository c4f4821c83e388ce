#!/bin/bash
# A/B of the in-tree library against paper_2303_10384_b200/lib/ab/*.so on the joint modes, 3 alternating reps.
O=gpurun_out/abj; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for rep in 1 2 3; do for cfg in c3 p124; do for m in joint joint_grad; do
  for lib in paper_2303_10384_b200/lib/librnnt_b200.so paper_2303_10384_b200/lib/ab/*.so; do
    n=$(basename $lib .so)
    RNNT_B200_LIB=$PWD/$lib timeout -s KILL 120 python bench.py --mode $m --config $cfg --steps 60 --no-cpu-baseline > $O/b.json 2>/dev/null
    python -c "import json; d=json.load(open('$O/b.json')); print('$cfg $m $n', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
  done; done; done; done > $O/summary.txt 2>&1
