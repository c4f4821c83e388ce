#!/bin/bash
# K3(c) on aux[c] right after K2(c) (RNNT_K3_ON_AUX=1) vs all K3 chunks on the caller's stream (default)
out=gpurun_out/k3aux.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
RNNT_K3_ON_AUX=1 timeout -s KILL 900 python -m pytest tests/test_parity.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/k3aux_pytest.log 2>&1
echo "aux pytest exit $? $(tail -1 gpurun_out/k3aux_pytest.log)" >> $out
for rep in 1 2 3; do for v in 1 0; do for c in "--config c2" "--config c3" "--config p124" "--config c3 --dtype bf16"; do
  RNNT_K3_ON_AUX=$v timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('aux=$v', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done; done
