#!/bin/bash
# K2 operand staging: cp.async shared-memory ring (default) vs round 1's register groups (RNNT_K2_REGSTAGE=1 build)
out=gpurun_out/k2ring.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_parity.py tests/test_canaries.py tests/test_viterbi.py tests/test_lattice.py -q -x -m gpu -p no:cacheprovider > gpurun_out/k2ring_pytest.log 2>&1
echo "pytest exit $?" >> $out; tail -2 gpurun_out/k2ring_pytest.log >> $out
for v in base k2reg; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  echo "== $v" >> $out
  RNNT_B200_LIB=$L timeout -s KILL 300 python scripts/k2_steps.py rnnt,allow_ignore >> $out 2>&1
done
for rep in 1 2; do for v in base k2reg; do for c in "--config c2" "--config c3" "--config p124" "--mode joint_grad --config p124"; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
