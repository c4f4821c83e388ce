#!/bin/bash
# K6 builders' tanh: RNNT_K6_NR of the 4 words per item with the reciprocal as Newton steps on the FMA pipe
# (working tree default = 2) vs 0 / 1 / 4 and HEAD (MUFU rcp for every word)
out=gpurun_out/k6nr.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 500 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/k6nr_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/k6nr_pytest.log)" >> $out
RNNT_B200_LIB=$PWD/paper_2303_10384_b200/lib/librnnt_b200_nr4.so timeout -s KILL 500 python -m pytest tests/test_joint.py -q -x -m gpu -p no:cacheprovider > gpurun_out/k6nr4_pytest.log 2>&1
echo "nr4 pytest exit $? $(tail -1 gpurun_out/k6nr4_pytest.log)" >> $out
for rep in 1 2; do for v in head nr0 nr1 base nr4; do for c in "--mode joint --config p124" "--mode joint --config c3" "--mode joint_grad --config p124" "--mode joint_grad --config c3"; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
