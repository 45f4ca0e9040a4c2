#!/bin/bash
# same-box A/B: k_colsT with bulk-staged P columns (working tree) vs without (nobulk)
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_configs.py -x -q > gpurun_out/ab8_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab8_tests.log
for round in 1 2; do
  for lib in notma new; do
    if [ $lib = new ]; then export RTN_LIB=$PWD/paper_1701_08361_b200/librtnlinv_b200.so; else export RTN_LIB=$PWD/build_var/lib_$lib.so; fi
    for c in c3 c4 c1; do timeout 120 python scripts/decomp_probe.py $c 3x1 | sed "s/^/$lib $c /"; done
    for c in c5 c2; do timeout 120 python scripts/decomp_probe.py $c 2x1 | sed "s/^/$lib $c /"; done
    RTN_CLUSTER=0 timeout 120 python scripts/decomp_probe.py c3 1x1 | sed "s/^/$lib c3-passes /"
    REPS=50 timeout 120 python scripts/prof_kernels.py c3 colsT | sed "s/^/$lib /"
  done
done > gpurun_out/ab8.txt 2>&1
