#!/bin/bash
# A/B of build_var/lib_base.so (committed tree) against the working tree's library on
# the default-schedule decomposition probes; run under gpurun
for n in base new base new; do
  if [ $n = base ]; then export RTN_LIB=$PWD/build_var/lib_base.so; else unset RTN_LIB; fi
  echo "== $n"
  timeout 100 python scripts/decomp_probe.py c3 3x1
  RTN_CLUSTER=0 timeout 100 python scripts/decomp_probe.py c3 1x1
  timeout 100 python scripts/decomp_probe.py c3 1x1
  timeout 100 python scripts/decomp_probe.py c4 3x1
  timeout 100 python scripts/decomp_probe.py c2 3x1
  timeout 100 python scripts/decomp_probe.py c1 3x1
done
