#!/bin/bash
# marginal cost of each pass in the running C3 T=3 mix (RTN_DOUBLE), the fixed cost of one
# more launch (nop), and the saturation point of independent slice series (five-kernel passes)
for d in none nop colsW rows1 colsT rows2; do
  RTN_DOUBLE=$d timeout 120 python scripts/decomp_probe.py ${CFG:-c3} 3x1 | sed "s/^/$d /"
done
RTN_SLICE_CLUSTER=0 timeout 300 python scripts/slices_probe.py 1 3 6
