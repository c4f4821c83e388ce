#!/bin/bash
# K6 forward with 16 builder warps (RNNT_K6_BUILDERS=16 build, 896 threads) vs 8 (base); joint parity of the variant
out=gpurun_out/b16.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
RNNT_B200_LIB=$PWD/paper_2303_10384_b200/lib/librnnt_b200_b16.so timeout -s KILL 300 python -m pytest tests/test_joint.py -q -x -m gpu -p no:cacheprovider -k "not many_short and not H384 and not H128 and not _128_ and not 384" > gpurun_out/b16_pytest.log 2>&1
echo "b16 pytest exit $? $(tail -1 gpurun_out/b16_pytest.log)" >> $out
for rep in 1 2; do for v in base b16; do for c in "--mode joint --config p124" "--mode joint --config c3" "--mode joint_grad --config p124" "--mode joint_grad --config c3"; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
