#!/bin/bash
# GPU tests, then the default-schedule probes with the deferred CR reductions on/off
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ab2_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab2_tests.log
for round in 1 2; do
  for dr in 1 0; do
    export RTN_DEFER_RED=$dr
    for c in c3 c4 c1; do timeout 120 python scripts/decomp_probe.py $c 3x1 | sed "s/^/defer$dr $c /"; done
    for c in c5 c2; do timeout 120 python scripts/decomp_probe.py $c 2x1 | sed "s/^/defer$dr $c /"; done
    RTN_CLUSTER=0 timeout 100 python scripts/decomp_probe.py c3 1x1 | sed "s/^/defer$dr c3-passes /"
  done
done > gpurun_out/ab2.txt 2>&1
REPS=50 timeout 300 python scripts/prof_kernels.py c3 colA rows1 colsT rows2 colsW cr_fused crA apply > gpurun_out/ab2_isolated.txt 2>&1
