#!/bin/bash
# same-box A/B: k_crA with a 2-block residency target (128 registers, spill-free)
for round in 1 2; do
  for lib in base cra2; do
    export RTN_LIB=$PWD/build_var/lib_$lib.so
    for c in c3 c4 c1; do timeout 120 python scripts/decomp_probe.py $c 3x1 | sed "s/^/$lib $c /"; done
    timeout 120 python scripts/decomp_probe.py c2 3x1 | sed "s/^/$lib c2 /"
    RTN_CLUSTER=0 timeout 120 python scripts/decomp_probe.py c3 1x1 | sed "s/^/$lib c3-passes /"
  done
done > gpurun_out/ab24.txt 2>&1
