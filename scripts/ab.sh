#!/bin/bash
# Same-box A/B of two builds of the library on the default-schedule probes (run under
# gpurun): A = $AB_A (default build_var/lib_base.so), B = $AB_B (default: the
# in-tree library of the working tree); AB_CFGS picks the throughput configs
A=${AB_A:-$PWD/build_var/lib_base.so}
B=${AB_B:-$PWD/paper_1701_08361_b200/librtnlinv_b200.so}
CFGS=${AB_CFGS:-"c3 c4 c1"}
for lib in "$A" "$B" "$A" "$B"; do
  export RTN_LIB=$lib
  echo "== $(basename $lib)"
  for c in $CFGS; do timeout 100 python scripts/decomp_probe.py $c 3x1 | sed "s/^/$c /"; done
  RTN_CLUSTER=0 timeout 100 python scripts/decomp_probe.py c3 1x1 | sed "s/^/c3-passes /"
  timeout 100 python scripts/decomp_probe.py c3 1x1 | sed "s/^/c3-latency /"
done
