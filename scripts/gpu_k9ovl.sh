#!/bin/bash
# K9 || K7 overlap: correctness, then the training step for several K9 SM caps.
O=gpurun_out/k9ovl; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 240 python -m pytest tests/test_joint.py tests/test_canaries.py -q -p no:cacheprovider -x --timeout 60 > $O/pytest_joint.log 2>&1; echo "exit $?" >> $O/pytest_joint.log
for cfg in c3 p124; do for n in 0 136 128 120 112 96; do
  RNNT_K9_CTAS=$n timeout -s KILL 120 python bench.py --mode joint_grad --config $cfg --steps 40 --warmup 5 --no-cpu-baseline > $O/b_${cfg}_$n.json 2>/dev/null
  python -c "import json; d=json.load(open('$O/b_${cfg}_$n.json')); print('$cfg', $n, round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done; done > $O/summary.txt 2>&1
echo done
