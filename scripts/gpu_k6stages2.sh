#!/bin/bash
# K6 / k6_dz_2sm W-stage count on the final tree: default (as many as fit) vs 4 / 6 / 8
out=gpurun_out/k6stages2.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do for st in def 4 6 8; do for c in "--mode joint --config p124" "--mode joint --config c3" "--mode joint_grad --config p124"; do
  if [ $st = def ]; then E=""; else E="RNNT_K6_STAGES=$st"; fi
  env $E timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('stages=$st', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
