#!/bin/bash
O=gpurun_out/san; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
which compute-sanitizer > $O/which.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_case.py > $O/$tool.log 2>&1
  echo "$tool exit $?" >> $O/summary.txt
done
