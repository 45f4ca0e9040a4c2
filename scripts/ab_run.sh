#!/bin/bash
# block-wide deferred partial sums in cr_begin (bsum) vs warp-0 sums (base); parity of bsum
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_ops.py tests/test_gpu_channel.py -x -q > gpurun_out/ab26_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab26_tests.log
for round in 1 2 3; do
  for v in base bsum; do
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c5 2x1 | sed "s/^/$v c5 /"
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c3 3x1 | sed "s/^/$v c3 /"
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c2 3x1 | sed "s/^/$v c2 /"
  done
done > gpurun_out/ab26.txt 2>&1
