#!/bin/bash
# C2 / C5 parity and the per-kernel factorisation defaults
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_ops.py -x -q -k "c2 or c5 or 320 or 384" > gpurun_out/ab23_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab23_tests.log
for round in 1 2; do
  timeout 120 python scripts/decomp_probe.py c5 2x1 | sed "s/^/c5 /"
  timeout 120 python scripts/decomp_probe.py c2 3x1 2x1 1x1 | sed "s/^/c2 /"
done > gpurun_out/ab23.txt 2>&1
