#!/bin/bash
# 16-bit K1: row pairs per warp 1 (base) / 2 / 4 (RNNT_K1_PAIRS builds), c3 bf16 and fp16 loss+grad; parity of each
out=gpurun_out/k1pairs.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for v in k1p2 k1p4; do
  RNNT_B200_LIB=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so timeout -s KILL 600 python -m pytest tests/test_parity_half.py -q -x -m gpu -p no:cacheprovider > gpurun_out/k1pairs_$v.log 2>&1
  echo "$v pytest exit $? $(tail -1 gpurun_out/k1pairs_$v.log)" >> $out
done
for rep in 1 2; do for v in base k1p2 k1p4; do for c in "--dtype bf16" "--dtype f16" "--dtype bf16 --mode loss"; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
