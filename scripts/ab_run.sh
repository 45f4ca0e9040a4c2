#!/bin/bash
# pass path knobs at T = 3: rho blocks of k_colsW / k_crA (RTN_RHO_BLOCKS, default clamp(L^2/512, 16, 148))
# and the k_cr_fused grid (RTN_VEC_BLOCKS, default min(D/1024, 296))
for round in 1 2; do
  for kv in "X=0" "RTN_RHO_BLOCKS=16" "RTN_RHO_BLOCKS=64" "RTN_RHO_BLOCKS=128" "RTN_VEC_BLOCKS=148" "RTN_VEC_BLOCKS=222"; do
    for c in c3 c4 c2; do
      env $kv timeout 120 python scripts/decomp_probe.py $c 3x1 | sed "s/^/$kv $c /"
    done
  done
done > gpurun_out/ab32.txt 2>&1
