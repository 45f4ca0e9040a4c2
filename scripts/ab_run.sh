#!/bin/bash
# C5 knobs: vector-recurrence grid and rho blocks; C3 vector grid
for round in 1 2; do
  timeout 120 python scripts/decomp_probe.py c5 2x1 | sed "s/^/c5 default /"
  for v in 444 592; do RTN_VEC_BLOCKS=$v timeout 120 python scripts/decomp_probe.py c5 2x1 | sed "s/^/c5 vec$v /"; done
  for r in 72 144; do RTN_RHO_BLOCKS=$r timeout 120 python scripts/decomp_probe.py c5 2x1 | sed "s/^/c5 rho$r /"; done
  RTN_CRA=1 timeout 120 python scripts/decomp_probe.py c5 2x1 | sed "s/^/c5 crA /"
  for v in 148 444; do RTN_VEC_BLOCKS=$v timeout 120 python scripts/decomp_probe.py c3 3x1 | sed "s/^/c3 vec$v /"; done
done > gpurun_out/ab12.txt 2>&1
