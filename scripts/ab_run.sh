#!/bin/bash
# latency mode (T = 1, cluster-fused applications): k_rho_sum grid size (RTN_RHO_SUM_BLOCKS; default min(L^2/32, 592))
for round in 1 2; do
  for nb in default 148 296 256 128; do
    for c in c3 c4 c1; do
      if [ $nb = default ]; then timeout 120 python scripts/decomp_probe.py $c 1x1 | sed "s/^/$nb $c /"
      else RTN_RHO_SUM_BLOCKS=$nb timeout 120 python scripts/decomp_probe.py $c 1x1 | sed "s/^/$nb $c /"; fi
    done
  done
done > gpurun_out/ab30.txt 2>&1
