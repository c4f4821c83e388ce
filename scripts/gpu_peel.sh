#!/bin/bash
# (the peeled K1 / K3 variant measured here was reverted: see DESIGN.md §10 and profiles/r02_g/peel_ab.txt)
# K1 / K3 on 16-bit rows with V % 8 == 4 as a 64-bit piece + 128-bit vectors (default) vs 64-bit vectors
# (RNNT_K3_PEEL=0): parity, bench lines, per-kernel times
out=gpurun_out/peel.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_parity_half.py tests/test_parity.py -q -x -m gpu -p no:cacheprovider > gpurun_out/peel_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/peel_pytest.log)" >> $out
for rep in 1 2; do for pe in 0 1; do for d in f16 bf16; do
  RNNT_K3_PEEL=$pe timeout -s KILL 200 python bench.py --config p124 --dtype $d --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('peel=$pe', '$d', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['roofline']['frac'], d['clocks']['sm_mhz'])" >> $out
done; done; done
for pe in 0 1; do
  RNNT_K3_PEEL=$pe timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k1_|k3_' -c 8 --csv --log-file gpurun_out/peel_ncu_$pe.csv python bench.py --config p124 --dtype f16 --steps 2 --warmup 3 --eager --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
