#!/bin/bash
O=gpurun_out/r02g; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
timeout -s KILL 400 python -m pytest tests/test_joint.py -q -p no:cacheprovider --timeout 120 -s -k "gemm_shapes or no_valid_rows or many_short" > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
