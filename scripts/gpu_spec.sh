#!/bin/bash
# K1 / K3 first chunk issued before the lengths (default, RNNT_SPEC_LOADS=1) vs length-gated (nospec build); parity first
out=gpurun_out/spec.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_parity.py tests/test_parity_half.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/spec_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/spec_pytest.log)" >> $out
for rep in 1 2; do for v in base nospec; do for c in "--config c2" "--config p124" "--config p124 --dtype f16" "--config c3" "--config c3 --dtype bf16" "--config c4 --variant allow_ignore"; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" >> $out
done; done; done
