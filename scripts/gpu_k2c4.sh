#!/bin/bash
# K2 for 65..128 columns: one warp x 4 columns per lane (RNNT_K2_CELLS=4) vs 4 warps x 1 column (default)
out=gpurun_out/k2c4.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
RNNT_K2_CELLS=4 timeout -s KILL 600 python -m pytest tests/test_parity.py -q -x -m gpu -p no:cacheprovider > gpurun_out/k2c4_pytest.log 2>&1
echo "cells=4 pytest exit $? $(tail -1 gpurun_out/k2c4_pytest.log)" >> $out
for v in 0 4; do echo "== cells=$v" >> $out; RNNT_K2_CELLS=$v timeout -s KILL 300 python scripts/k2_steps.py rnnt >> $out 2>&1; done
for rep in 1 2; do for v in 0 4; do for c in "--mode joint_grad --config p124" "--mode joint_grad --config c3" "--config p124"; do
  RNNT_K2_CELLS=$v timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('cells=$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
