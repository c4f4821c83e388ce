#!/bin/bash
O=gpurun_out/longu; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
RNNT_MARGINS_OUT=$O/margins.jsonl timeout -s KILL 900 python -m pytest tests/test_parity.py tests/test_viterbi.py tests/test_joint.py -q -p no:cacheprovider --timeout 300 > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
