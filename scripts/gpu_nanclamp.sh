#!/bin/bash
# Newton tanh's clamp as compare + select (NaN-propagating) vs fminf (HEAD): NaN test, joint tests, p124 / c3 joint
out=gpurun_out/nanclamp.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_joint.py -q -x -m gpu -p no:cacheprovider > gpurun_out/nanclamp_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/nanclamp_pytest.log)" >> $out
RNNT_B200_LIB=$PWD/paper_2303_10384_b200/lib/librnnt_b200_head.so timeout -s KILL 300 python -m pytest tests/test_joint.py -q -m gpu -p no:cacheprovider -k nan > gpurun_out/nanclamp_head.log 2>&1
echo "head nan test exit $? $(tail -1 gpurun_out/nanclamp_head.log)" >> $out
for rep in 1 2 3; do for v in head base; do for c in p124 c3; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py --mode joint --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
