#!/bin/bash
# Full GPU suite (tanh.approx builders) + the joint benches.
O=gpurun_out/r02f; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
RNNT_MARGINS_OUT=$O/margins.jsonl timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -s > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
for m in joint joint_grad; do for cfg in c3 p124; do
timeout -s KILL 200 python bench.py --mode $m --config $cfg --no-cpu-baseline > $O/bench_${m}_$cfg.json 2> $O/bench_${m}_$cfg.err; done; done
echo done
