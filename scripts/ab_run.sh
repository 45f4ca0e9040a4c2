#!/bin/bash
# latency-mode knobs: k_rho_sum grid and the vector-recurrence grid at T = 1
for round in 1 2; do
  for r in 512 256 148; do RTN_RHO_SUM_BLOCKS=$r timeout 120 python scripts/decomp_probe.py c3 1x1 | sed "s/^/rhosum$r /"; done
  for v in 148 296 444; do RTN_VEC_BLOCKS=$v timeout 120 python scripts/decomp_probe.py c3 1x1 | sed "s/^/vec$v /"; done
done > gpurun_out/ab19.txt 2>&1
