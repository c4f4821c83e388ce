#!/bin/bash
# Round 2, first check: all GPU tests (parity margins logged), smoke(), the default bench line, a two-rank
# self-launched bench over gloo on the one GPU, the joint training step, and the launch list of bench.py.
O=gpurun_out/r02a; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
RNNT_MARGINS_OUT=$O/margins.jsonl timeout -s KILL 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -s > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout -s KILL 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout -s KILL 900 python bench.py --gpus 2 --backend gloo --scaling strong --no-e2e --no-cpu-baseline > $O/bench_c3_gloo2_strong.json 2> $O/bench_c3_gloo2_strong.err
timeout -s KILL 900 python bench.py --mode joint_grad --no-cpu-baseline > $O/bench_joint_grad_c3.json 2> $O/bench_joint_grad_c3.err
timeout -s KILL 900 python bench.py --mode joint_grad --config p124 --no-cpu-baseline > $O/bench_joint_grad_p124.json 2> $O/bench_joint_grad_p124.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --eager > $O/ncu.log 2>&1
echo done
