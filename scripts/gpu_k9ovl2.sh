#!/bin/bash
O=gpurun_out/k9ovl2; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for rep in 1 2 3; do for cfg in c3 p124; do for n in 0 96 112; do
  RNNT_K9_CTAS=$n timeout -s KILL 120 python bench.py --mode joint_grad --config $cfg --steps 60 --warmup 5 --no-cpu-baseline > $O/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b.json')); print('$cfg', $n, round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done; done > $O/summary.txt 2>&1
