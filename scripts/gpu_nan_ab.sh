#!/bin/bash
# (first run: the NaN map with a per-word check cost bf16 c3 K1 0.740 -> 0.777 ms through extra local-memory traffic; this run: the lse-only check, parity with the previous library)
# NaN semantics change (Populate maps NaN arc scores to +inf, K2 reports log P = +inf as NaN, Newton clamp by
# select) vs the library before it (head): same box, alternating
out=gpurun_out/nan_ab.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_parity.py tests/test_joint.py tests/test_parity_half.py -q -m gpu -p no:cacheprovider -k "nan or half_random" > gpurun_out/nan_ab_pytest.log 2>&1; echo "pytest exit $? $(tail -1 gpurun_out/nan_ab_pytest.log)" >> $out
for rep in 1 2 3; do for v in head base; do for c in "--config c3" "--config c3 --dtype bf16" "--config p124 --dtype f16"; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
