#!/bin/bash
# K8 drain: 32-column TMEM loads (RNNT_K8_LD32=1 build) vs 16-column (base); parity of the variant, A/B, K8 roles
out=gpurun_out/k8ld32.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_ld32.so
RNNT_B200_LIB=$L timeout -s KILL 400 python -m pytest tests/test_joint.py -q -x -m gpu -p no:cacheprovider -k "grad" > gpurun_out/k8ld32_pytest.log 2>&1
echo "ld32 pytest exit $? $(tail -1 gpurun_out/k8ld32_pytest.log)" >> $out
for rep in 1 2 3; do for v in base ld32; do for c in p124 c3; do
  if [ $v = base ]; then LL=""; else LL=$L; fi
  RNNT_B200_LIB=$LL timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done; done
for v in base ld32; do for c in p124 c3; do
  if [ $v = base ]; then LL=""; else LL=$L; fi
  echo "$v $c $(RNNT_B200_LIB=$LL RNNT_K8_DEBUG=4 timeout -s KILL 120 python bench.py --mode joint_grad --config $c --steps 1 --warmup 3 --eager --no-cpu-baseline --no-e2e 2>&1 | grep 'K8 pair' | tail -1)" >> $out
done; done
