#!/bin/bash
# Round-2 evidence: all GPU tests (margins logged), smoke(), one bench line per mode / config, launch lists and
# ncu captures of the training step's new kernels.
O=gpurun_out/final11; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
RNNT_MARGINS_OUT=$O/margins.jsonl timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -s > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
run() { name=$1; shift; timeout -s KILL 600 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; }
t0=$(date +%s); timeout -s KILL 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "$(( $(date +%s) - t0 )) s wall (default bench.py)" > $O/bench_c3.walltime
run c3_bf16 --dtype bf16 --no-cpu-baseline
run c2 --config c2 --no-e2e --no-cpu-baseline
run c4ff --config c4 --variant force_final --no-e2e --no-cpu-baseline
run c4ai --config c4 --variant allow_ignore --no-e2e --no-cpu-baseline
run c3_loss --mode loss --no-e2e --no-cpu-baseline
run c3_viterbi --mode viterbi --no-e2e --no-cpu-baseline
run c3_lattice --mode lattice --no-e2e --no-cpu-baseline
run joint_c3 --mode joint
run joint_p124 --mode joint --config p124 --no-cpu-baseline
run joint_grad_c3 --mode joint_grad --no-cpu-baseline
run joint_grad_p124 --mode joint_grad --config p124 --no-cpu-baseline
run c5 --config c5 --no-e2e --no-cpu-baseline --steps 10 --warmup 3
run p124 --config p124 --no-e2e
run p124_f16 --config p124 --dtype f16 --no-e2e --no-cpu-baseline
run c3_gloo2_strong --gpus 2 --backend gloo --scaling strong --no-e2e --no-cpu-baseline
timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 3 --eager --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_joint_grad_c3.csv python bench.py --mode joint_grad --steps 2 --warmup 3 --eager --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_joint_grad_p124.csv python bench.py --mode joint_grad --config p124 --steps 2 --warmup 3 --eager --no-cpu-baseline > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:'k6_dz|k6_joint|k8_dh' -s 3 -c 3 -o $O/k68_full python bench.py --mode joint_grad --steps 1 --warmup 1 --eager --no-cpu-baseline > $O/ncu_full.log 2>&1
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:'k6_joint' -c 1 -o $O/k6_p124_full python bench.py --mode joint --config p124 --steps 1 --warmup 1 --eager --no-cpu-baseline --no-e2e > $O/ncu_k6_p124.log 2>&1
echo done
