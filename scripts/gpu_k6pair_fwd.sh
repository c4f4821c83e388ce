#!/bin/bash
# K6 forward: pair MMAs (default) vs per-CTA MMAs with W multicast (RNNT_K6_PAIR=0), p124 / c3, joint + training
out=gpurun_out/k6pairfwd.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2 3; do for v in 1 0; do for c in "--mode joint --config p124" "--mode joint --config c3" "--mode joint_grad --config p124"; do
  RNNT_K6_PAIR=$v timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('pair=$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
