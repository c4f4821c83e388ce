#!/bin/bash
# K7 with 16 frames per block (default) vs 8 (RNNT_K7_FRAMES=8 build): joint parity, training-step A/B, launch lists
out=gpurun_out/k7f16.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 400 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/k7f16_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/k7f16_pytest.log)" >> $out
for rep in 1 2 3; do for v in base f8; do for c in p124 c3; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done; done
O=gpurun_out/k7l; mkdir -p $O
for v in base f8; do for cfg in p124 c3; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
  RNNT_B200_LIB=$L timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/l_${v}_$cfg.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 3 --eager --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "$v $cfg"; python scripts/launch_summary.py $O/l_${v}_$cfg.csv | grep -E "k7_"; done; done > $O/summary.txt 2>&1
