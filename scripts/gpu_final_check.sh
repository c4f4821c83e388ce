#!/bin/bash
# last check of the final tree: every GPU test, smoke(), the default bench line and the Viterbi line
O=gpurun_out/final12; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout -s KILL 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout -s KILL 600 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout -s KILL 300 python bench.py --mode viterbi --no-e2e --no-cpu-baseline > $O/bench_c3_viterbi.json 2> $O/bench_c3_viterbi.err
