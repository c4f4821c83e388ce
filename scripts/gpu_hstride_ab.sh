#!/bin/bash
# A/B of the aligned h stride: the in-tree library vs lib/ab/librnnt_b200_old.so (the previous commit built and
# copied there by hand; git-ignored), joint training step c3 / p124, 3 alternating reps, plus the joint parity tests.
mkdir -p gpurun_out/hs
timeout -s KILL 600 python -m pytest tests/test_joint.py tests/test_canaries.py -m gpu -q -p no:cacheprovider > gpurun_out/hs/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/hs/pytest.log
for rep in 1 2 3; do
  for lib in paper_2303_10384_b200/lib/librnnt_b200.so paper_2303_10384_b200/lib/ab/librnnt_b200_old.so; do
    n=$(basename $lib .so)
    for cfg in c3 p124; do
      RNNT_B200_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --mode joint_grad --config $cfg --no-e2e \
        --no-cpu-baseline > gpurun_out/hs/${n}_${cfg}_$rep.json 2>/dev/null
    done
  done
done
