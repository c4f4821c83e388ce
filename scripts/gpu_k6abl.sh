#!/bin/bash
mkdir -p gpurun_out; rm -f gpurun_out/k6abl.txt
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for cfg in "--config p124" ""; do
for d in 0 1 2 3; do
  RNNT_K6_DEBUG=$d timeout -s KILL 200 python bench.py --mode joint $cfg --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('dbg=$d', '$cfg', round(d['value']), round(d['kernels_ms']['k6_joint_lse'],4), d['clocks']['sm_mhz'])" >> gpurun_out/k6abl.txt
done; done
