#!/bin/bash
# All GPU tests + smoke + the joint training-step bench lines (c3, p124) on one box.
mkdir -p gpurun_out/chk
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/chk/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/chk/pytest_gpu.log
timeout -s KILL 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/chk/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/chk/smoke.log
timeout -s KILL 300 python bench.py --mode joint_grad --no-cpu-baseline > gpurun_out/chk/bench_joint_grad_c3.json 2> gpurun_out/chk/bench_joint_grad_c3.err
timeout -s KILL 300 python bench.py --mode joint_grad --config p124 --no-cpu-baseline > gpurun_out/chk/bench_joint_grad_p124.json 2> gpurun_out/chk/bench_joint_grad_p124.err
