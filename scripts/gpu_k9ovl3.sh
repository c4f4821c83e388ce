#!/bin/bash
# K9 beside K7 (K9 capped at n SMs on a high-priority stream, K7 on the rest) vs sequential (0), current tree
out=gpurun_out/k9ovl3.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2 3; do for n in 0 96 112 128; do for c in p124 c3; do
  RNNT_K9_CTAS=$n timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('k9_ctas=$n', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done; done
