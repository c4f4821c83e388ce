#!/bin/bash
O=gpurun_out/abk1; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for rep in 1 2 3; do for lib in paper_2303_10384_b200/lib/librnnt_b200.so paper_2303_10384_b200/lib/ab/*.so; do
    n=$(basename $lib .so)
    RNNT_B200_LIB=$PWD/$lib timeout -s KILL 120 python bench.py --dtype bf16 --no-e2e --no-cpu-baseline > $O/b.json 2>/dev/null
    python -c "import json; d=json.load(open('$O/b.json')); print('$n', round(d['ms_per_step'],4), round(d['kernels_ms']['k1_lse_gather'],4), d['clocks']['sm_mhz'])"
done; done > $O/summary.txt 2>&1
