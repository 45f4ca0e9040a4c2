#!/bin/bash
# k_cr_fused<false> + crA without the group branch + block-wide group member sums (new) vs HEAD (base)
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_ops.py tests/test_gpu_channel.py tests/test_gpu_procgroup.py -x -q > gpurun_out/ab28_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab28_tests.log
for round in 1 2 3; do
  for v in base new; do
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c3 3x1 1x1 1x2 | sed "s/^/$v c3 /"
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c4 3x1 | sed "s/^/$v c4 /"
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c2 3x1 | sed "s/^/$v c2 /"
  done
done > gpurun_out/ab28.txt 2>&1
