#!/bin/bash
# A/B of the persistent iteration kernel (k_flow) against the five pass kernels +
# k_cr_fused on the same box: correctness of the default build first, then C3/C4
# throughput (T = 3) and T = 1 five-kernel-class latency for every build_var variant.
timeout 600 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_configs.py -k "c3_bench or c4_T8 or c2_bench" 2>&1 | tail -3
for lib in build_var/lib_*.so; do
  export RTN_LIB=$PWD/$lib
  for flow in 1 0; do
    [ "$flow" = 0 ] && [ "$lib" != "build_var/lib_noi3.so" ] && continue
    echo "== $(basename $lib) RTN_FLOW=$flow"
    for c in ${FLOW_CFGS:-c3 c4}; do RTN_FLOW=$flow timeout 100 python scripts/decomp_probe.py $c 3x1 | sed "s/^/$c /"; done
    RTN_FLOW=$flow RTN_CLUSTER=0 timeout 100 python scripts/decomp_probe.py c3 1x1 | sed "s/^/c3-passes /"
  done
done
