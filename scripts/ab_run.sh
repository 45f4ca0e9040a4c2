#!/bin/bash
# k_colsT with its P entries loaded before the exchange (prep) vs after step 2 (base); parity of prep
RTN_LIB=build_var/lib_prep.so timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_ops.py -x -q > gpurun_out/ab29_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab29_tests.log
for round in 1 2 3; do
  for v in base prep; do
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c3 3x1 1x1 | sed "s/^/$v c3 /"
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c4 3x1 | sed "s/^/$v c4 /"
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c2 3x1 | sed "s/^/$v c2 /"
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c5 2x1 | sed "s/^/$v c5 /"
    RTN_LIB=build_var/lib_$v.so timeout 120 python scripts/decomp_probe.py c1 3x1 | sed "s/^/$v c1 /"
  done
done > gpurun_out/ab29.txt 2>&1
