#!/bin/bash
# fused small-call schedule (default where eligible) vs the chunked one (RNNT_FUSED=0): parity, A/B, launch list
out=gpurun_out/fused.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_parity.py tests/test_canaries.py tests/test_dist_gpu.py tests/test_parity_half.py -q -x -m gpu -p no:cacheprovider > gpurun_out/fused_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/fused_pytest.log)" >> $out
for rep in 1 2 3; do for v in 1 0; do for c in "--config c2" "--config c2 --mode loss" "--config c3"; do
  RNNT_FUSED=$v timeout -s KILL 120 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('fused=$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
