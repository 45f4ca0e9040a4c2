#!/bin/bash
# Same-box A/B of two library builds in latency mode (T = 1, cluster-fused where the
# grid has it); A = $AB_A (default build_var/lib_base.so), B = $AB_B (default: in-tree)
A=${AB_A:-$PWD/build_var/lib_base.so}
B=${AB_B:-$PWD/paper_1701_08361_b200/librtnlinv_b200.so}
for lib in "$A" "$B" "$A" "$B"; do
  export RTN_LIB=$lib
  echo "== $(basename $lib)"
  timeout 100 python scripts/decomp_probe.py c3 1x1
  timeout 100 python scripts/decomp_probe.py c4 1x1
  timeout 100 python scripts/decomp_probe.py c1 1x1
done
