#!/bin/bash
# bf16 widening as PRMT (RNNT_BF16_PRMT=1 build) vs the default shift (IMAD.U32): c3 / p124 bf16 loss+grad, parity
out=gpurun_out/prmt.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
RNNT_B200_LIB=$PWD/paper_2303_10384_b200/lib/librnnt_b200_prmt.so timeout -s KILL 600 python -m pytest tests/test_parity_half.py tests/test_joint.py -q -x -m gpu -p no:cacheprovider > gpurun_out/prmt_pytest.log 2>&1
echo "prmt pytest exit $? $(tail -1 gpurun_out/prmt_pytest.log)" >> $out
for rep in 1 2 3; do for v in base prmt; do for c in "--dtype bf16" "--dtype bf16 --mode loss" "--dtype bf16 --config p124" "--mode joint_grad --config p124"; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
