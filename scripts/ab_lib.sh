#!/bin/bash
# A/B of the in-tree library vs a variant (lib/librnnt_b200_$VAR.so) on bench lines ($CASES: ';'-separated arg sets)
mkdir -p gpurun_out; rm -f gpurun_out/ab_lib.txt
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || exit 1
IFS=';' read -ra CS <<< "$CASES"
for rep in 1 2; do
  for v in base $VAR; do
    for c in "${CS[@]}"; do
      if [ $v = base ]; then L=""; else L=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$v.so; fi
      RNNT_B200_LIB=$L timeout -s KILL 200 python bench.py $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$c', round(d['value']), d['ms_per_step'], {k: round(x, 4) for k, x in d['kernels_ms'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/ab_lib.txt
    done
  done
done
if [ -n "$TESTS" ]; then
  RNNT_B200_LIB=$PWD/paper_2303_10384_b200/lib/librnnt_b200_$VAR.so timeout -s KILL 600 python -m pytest $TESTS -q -x -p no:cacheprovider > gpurun_out/ab_lib_pytest.log 2>&1
  echo "exit $?" >> gpurun_out/ab_lib_pytest.log
fi
