#!/bin/bash
# same-box A/B of library builds: base = build_var/lib_base.so (previous commit), new = the
# working tree's library, and the build_var variants named in AB_VARS
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_configs.py tests/test_gpu_series.py tests/test_gpu_channel.py tests/test_gpu_properties.py -x -q > gpurun_out/ab4_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab4_tests.log
for round in 1 2; do
  for lib in base new ${AB_VARS}; do
    if [ $lib = new ]; then export RTN_LIB=$PWD/paper_1701_08361_b200/librtnlinv_b200.so; else export RTN_LIB=$PWD/build_var/lib_$lib.so; fi
    for c in c3 c4 c1; do timeout 120 python scripts/decomp_probe.py $c 3x1 | sed "s/^/$lib $c /"; done
    for c in c5 c2; do timeout 120 python scripts/decomp_probe.py $c 2x1 | sed "s/^/$lib $c /"; done
    timeout 120 python scripts/decomp_probe.py c3 1x1 | sed "s/^/$lib c3-latency /"
  done
done > gpurun_out/ab4.txt 2>&1
