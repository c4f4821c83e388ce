#!/bin/bash
# K6 forward / training step vs the number of W stages (smaller shared memory -> larger L1 for the builders)
out=gpurun_out/k6stages.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do for st in 16 8 6 4 3; do for m in joint joint_grad; do for c in p124 c3; do
RNNT_K6_STAGES=$st timeout -s KILL 200 python bench.py --mode $m --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('stages=$st', '$m', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done; done
