#!/bin/bash
# Same-box A/B of several library builds (run under gpurun): AB_LIBS="base minb4 ..." names
# build_var/lib_<name>.so; AB_CFGS picks the configs, AB_PAIRS the (T x A) points
LIBS=${AB_LIBS:-"base"}
CFGS=${AB_CFGS:-"c3 c4 c1"}
PAIRS=${AB_PAIRS:-"3x1"}
for round in 1 2; do
  for name in $LIBS; do
    export RTN_LIB=$PWD/build_var/lib_$name.so
    for c in $CFGS; do timeout 120 python scripts/decomp_probe.py $c $PAIRS | sed "s/^/$name $c /"; done
  done
done
