#!/bin/bash
# K6 forward: bias-prefilled accumulators (default) vs the epilogue's bias add (RNNT_K6_DEBUG=128); and k6_dz_2sm's
# row-scalar lookahead re-checked (64) now that the A/B bits keep the forward builders' fast path
out=gpurun_out/prefill.txt; rm -f $out; mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout -s KILL 400 python -m pytest tests/test_joint.py tests/test_canaries.py -q -x -m gpu -p no:cacheprovider > gpurun_out/prefill_pytest.log 2>&1
echo "pytest exit $? $(tail -1 gpurun_out/prefill_pytest.log)" >> $out
for rep in 1 2 3; do for v in 0 128 64; do for c in "--mode joint --config c3" "--mode joint --config p124" "--mode joint_grad --config c3" "--mode joint_grad --config p124"; do
  RNNT_K6_DEBUG=$v timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('dbg=$v', '$c', round(d['value']), round(d['ms_per_step'],4), {k: round(x,4) for k,x in d.get('kernels_ms',{}).items()}, d['clocks']['sm_mhz'])" >> $out
done; done; done
for v in 4 132; do for c in p124 c3; do
  echo "dbg=$v $c $(RNNT_K6_DEBUG=$v timeout -s KILL 120 python bench.py --mode joint --config $c --steps 1 --warmup 3 --eager --no-cpu-baseline --no-e2e 2>&1 | grep 'K6 cycles' | tail -1)" >> $out
done; done
