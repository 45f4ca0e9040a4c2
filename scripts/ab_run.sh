#!/bin/bash
# latency mode: k_rho_sum 16-entry tiles (t16: half-warp channel groups, twice the blocks) vs 32 (t32); parity of t16
RTN_LIB=build_var/lib_t16.so timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_ops.py tests/test_gpu_channel.py -x -q > gpurun_out/ab31_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab31_tests.log
for round in 1 2 3; do
  for v in t32 t16; do
    for c in c3 c4 c1; do
      RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py $c 1x1 | sed "s/^/$v $c /"
    done
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c3 3x1 | sed "s/^/$v c3 /"
  done
done > gpurun_out/ab31.txt 2>&1
