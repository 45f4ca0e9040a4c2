#!/bin/bash
# Same-box A/B of two builds of the library on the default-schedule probes (run under
# gpurun): A = $AB_A (default build_var/lib_base.so), B = $AB_B (default: the
# in-tree library of the working tree)
A=${AB_A:-$PWD/build_var/lib_base.so}
B=${AB_B:-$PWD/paper_1701_08361_b200/librtnlinv_b200.so}
for lib in "$A" "$B" "$A" "$B"; do
  export RTN_LIB=$lib
  echo "== $(basename $lib)"
  timeout 100 python scripts/decomp_probe.py c3 3x1
  RTN_CLUSTER=0 timeout 100 python scripts/decomp_probe.py c3 1x1
  timeout 100 python scripts/decomp_probe.py c3 1x1
  timeout 100 python scripts/decomp_probe.py c4 3x1
  timeout 100 python scripts/decomp_probe.py c1 3x1
done
