#!/bin/bash
# Viterbi / lattice iteration: their GPU tests + bench lines for the alternate modes.
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_viterbi.py tests/test_canaries.py tests/test_lattice.py -q -x -p no:cacheprovider > gpurun_out/pytest_vit.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_vit.log
for v in rnnt force_final allow_ignore; do
  timeout 600 python bench.py --mode viterbi --variant $v --no-e2e --no-cpu-baseline > gpurun_out/bench_vit_$v.json 2> gpurun_out/bench_vit_$v.err
done
timeout 600 python bench.py --mode viterbi --config c5 --no-e2e --no-cpu-baseline > gpurun_out/bench_vit_c5.json 2> gpurun_out/bench_vit_c5.err
timeout 600 python bench.py --mode lattice --no-e2e --no-cpu-baseline > gpurun_out/bench_lat.json 2> gpurun_out/bench_lat.err
