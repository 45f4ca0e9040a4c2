#!/bin/bash
# same-box A/B: deferred reductions on the cluster (latency-mode) path
timeout 1500 python -m pytest tests/test_gpu_ops.py tests/test_gpu_series.py tests/test_gpu_configs.py -x -q -k "cluster or latency or g256 or c3 or c1 or c4" > gpurun_out/ab18_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab18_tests.log
for round in 1 2; do
  for lib in base new; do
    if [ $lib = new ]; then export RTN_LIB=$PWD/paper_1701_08361_b200/librtnlinv_b200.so; else export RTN_LIB=$PWD/build_var/lib_$lib.so; fi
    for c in c3 c4 c1; do timeout 120 python scripts/decomp_probe.py $c 1x1 3x1 | sed "s/^/$lib $c /"; done
  done
done > gpurun_out/ab18.txt 2>&1
