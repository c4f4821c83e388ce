#!/bin/bash
# k6_dz_2sm: dz through TMA tile stores (default) vs per-lane stores (RNNT_K6_DEBUG=32); joint parity first
mkdir -p gpurun_out; out=gpurun_out/dzstore.txt; rm -f $out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/dzstore_pytest.log 2>&1
echo "pytest exit $?" >> $out; tail -2 gpurun_out/dzstore_pytest.log >> $out
for rep in 1 2; do for d in 0 32; do for c in p124 c3; do
RNNT_K6_DEBUG=$d timeout -s KILL 200 python bench.py --mode joint_grad --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('dbg=$d', '$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])" >> $out
done; done; done
O=gpurun_out/dzs; mkdir -p $O
for d in 0 32; do
RNNT_K6_DEBUG=$d timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c3_$d.csv python bench.py --mode joint_grad --config c3 --steps 2 --warmup 3 --eager --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo "dbg=$d"; python scripts/launch_summary.py $O/launches_c3_$d.csv | grep -E "k6_dz|k6_joint"; done > $O/summary.txt 2>&1
