#!/bin/bash
# End-of-round evidence: all GPU tests, smoke(), and one bench line per mode / config.
mkdir -p gpurun_out/final
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/final/build.log 2>&1 || exit 1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/final/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/final/pytest_gpu.log
timeout -s KILL 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/final/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/final/smoke.log
run() { name=$1; shift; timeout -s KILL 900 python bench.py "$@" > gpurun_out/final/bench_$name.json 2> gpurun_out/final/bench_$name.err; }
t0=$(date +%s); timeout -s KILL 900 python bench.py > gpurun_out/final/bench_c3.json 2> gpurun_out/final/bench_c3.err; echo "$(( $(date +%s) - t0 )) s wall (default bench.py)" > gpurun_out/final/bench_c3.walltime
run c3_bf16 --dtype bf16 --no-e2e --no-cpu-baseline
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
run c3ff_lattice_compose --mode lattice --lattice compose --variant force_final --no-e2e --no-cpu-baseline
timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
