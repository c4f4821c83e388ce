#!/bin/bash
O=gpurun_out/host; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_parity.py -k "host or loss_sum" tests/test_abi.py -q -p no:cacheprovider --timeout 120 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout -s KILL 300 python bench.py --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
timeout -s KILL 300 python bench.py --dtype bf16 --no-cpu-baseline > $O/bench_c3_bf16.json 2> $O/bench_c3_bf16.err
echo done
