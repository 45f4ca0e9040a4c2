#!/bin/bash
# same-box A/B: deferred-total loads batched four per lane
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_channel.py -x -q -k "deferred or c3 or c1 or cluster" > gpurun_out/ab21_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab21_tests.log
for round in 1 2; do
  for lib in base new; do
    if [ $lib = new ]; then export RTN_LIB=$PWD/paper_1701_08361_b200/librtnlinv_b200.so; else export RTN_LIB=$PWD/build_var/lib_$lib.so; fi
    for c in c3 c4 c1; do timeout 120 python scripts/decomp_probe.py $c 1x1 3x1 | sed "s/^/$lib $c /"; done
    for c in c5 c2; do timeout 120 python scripts/decomp_probe.py $c 2x1 | sed "s/^/$lib $c /"; done
    REPS=50 timeout 120 python scripts/prof_kernels.py c3 cr_fused crA | sed "s/^/$lib /"
  done
done > gpurun_out/ab21.txt 2>&1
