#!/bin/bash
# same-box A/B: base (previous commit) vs the working tree (state flags loaded with the first operands)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab15_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab15_tests.log
for round in 1 2; do
  for lib in base new; do
    if [ $lib = new ]; then export RTN_LIB=$PWD/paper_1701_08361_b200/librtnlinv_b200.so; else export RTN_LIB=$PWD/build_var/lib_$lib.so; fi
    for c in c3 c4 c1; do timeout 120 python scripts/decomp_probe.py $c 3x1 | sed "s/^/$lib $c /"; done
    for c in c5 c2; do timeout 120 python scripts/decomp_probe.py $c 2x1 | sed "s/^/$lib $c /"; done
    timeout 120 python scripts/decomp_probe.py c3 1x1 | sed "s/^/$lib c3-latency /"
    RTN_CLUSTER=0 timeout 120 python scripts/decomp_probe.py c3 1x1 | sed "s/^/$lib c3-passes /"
    REPS=50 timeout 120 python scripts/prof_kernels.py c3 colA rows1 colsT rows2 colsW | sed "s/^/$lib /"
  done
done > gpurun_out/ab15.txt 2>&1
