#!/bin/bash
# K6 forward ablations at p124 / c3 (RNNT_K6_DEBUG): 0 none, 1 no tanh, 16 no f/g loads, 17 neither, 2 no epilogue math
out=gpurun_out/k6abl2.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for rep in 1 2; do for d in 0 1 16 17 2 18; do for c in p124 c3; do
RNNT_K6_DEBUG=$d timeout -s KILL 200 python bench.py --mode joint --config $c --no-e2e --no-cpu-baseline --steps 30 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('dbg=$d', '$c', {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
