#!/bin/bash
# channel groups after the deferred back-half partials: tests and single-GPU T x A probes
timeout 900 python -m pytest tests/test_gpu_channel.py tests/test_gpu_procgroup.py tests/test_gpu_series.py -x -q > gpurun_out/ab13_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab13_tests.log
for c in c3 c1 c4; do timeout 200 python scripts/decomp_probe.py $c 1x1 1x2 1x4 3x2 | sed "s/^/$c /"; done > gpurun_out/ab13.txt 2>&1
RTN_SERIES_CLUSTER=0 timeout 200 python scripts/decomp_probe.py c3 1x1 1x2 | sed "s/^/c3 passes /" >> gpurun_out/ab13.txt 2>&1
