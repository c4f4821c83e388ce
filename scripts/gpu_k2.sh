#!/bin/bash
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/k2_sweep.py c3 rnnt,force_final > gpurun_out/k2_sweep.json 2>&1
timeout 300 python scripts/k2_sweep.py c2 rnnt > gpurun_out/k2_sweep_c2.json 2>&1
