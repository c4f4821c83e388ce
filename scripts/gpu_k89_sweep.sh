#!/bin/bash
# K8 / K9 variants (cluster shapes) timed by ncu's launch list (cold, serialised: relative comparison only).
O=gpurun_out/k89sweep; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || exit 1
for cfg in c3 p124; do
for v in "RNNT_K8_RT=4 RNNT_K9_CLUSTER=8" "RNNT_K8_RT=2 RNNT_K9_CLUSTER=4" "RNNT_K8_RT=1 RNNT_K9_CLUSTER=2" "RNNT_K9_CLUSTER=1"; do
  tag=$(echo $v | tr ' =' '__')
  env $v timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k8_dh|k9_dw' -c 6 --csv --log-file $O/${cfg}_$tag.csv python bench.py --mode joint_grad --config $cfg --steps 2 --warmup 2 --eager --no-cpu-baseline > /dev/null 2>&1
  echo "$cfg $v"; python scripts/launch_summary.py $O/${cfg}_$tag.csv
done; done > $O/summary.txt 2>&1
echo done
