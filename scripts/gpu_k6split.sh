#!/bin/bash
# K6 per-role barrier-wait cycle split (RNNT_K6_DEBUG=4) for the forward and the training step, c3 and p124.
mkdir -p gpurun_out; rm -f gpurun_out/k6split.txt
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
for m in joint joint_grad; do for c in c3 p124; do
  echo "== $m $c" >> gpurun_out/k6split.txt
  RNNT_K6_DEBUG=4 timeout -s KILL 300 python bench.py --mode $m --config $c --no-e2e --no-cpu-baseline --steps 2 --warmup 3 --eager 2>&1 >/dev/null | grep "K6 cycles" | tail -2 >> gpurun_out/k6split.txt
done; done
