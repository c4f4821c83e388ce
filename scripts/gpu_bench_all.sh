#!/bin/bash
# Tests + the bench line for every BASELINE config that fits one GPU (c2, c3, c4 FF/AI, c5 shard).
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
if [ -z "$NO_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --config c2 --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --config c4 --variant force_final --no-e2e --no-cpu-baseline > gpurun_out/bench_c4ff.json 2> gpurun_out/bench_c4ff.err
timeout 600 python bench.py --config c4 --variant allow_ignore --no-e2e --no-cpu-baseline > gpurun_out/bench_c4ai.json 2> gpurun_out/bench_c4ai.err
timeout 900 python bench.py --config c5 --steps 20 --warmup 3 --cpu-threads 4 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
