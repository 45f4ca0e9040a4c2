#!/bin/bash
# channel-chunked applications (RTN_CHUNKS): C5 and C3 throughput, parity at C5 chunked
RTN_CHUNKS=2 timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_ops.py -x -q -k "c5 or c3_bench or 384" > gpurun_out/ab25_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab25_tests.log
for round in 1 2; do
  for ch in 1 2 4; do
    RTN_CHUNKS=$ch timeout 120 python scripts/decomp_probe.py c5 2x1 1x1 | sed "s/^/chunks$ch c5 /"
    RTN_CHUNKS=$ch timeout 120 python scripts/decomp_probe.py c3 3x1 | sed "s/^/chunks$ch c3 /"
    RTN_CHUNKS=$ch timeout 120 python scripts/decomp_probe.py c2 3x1 | sed "s/^/chunks$ch c2 /"
  done
done > gpurun_out/ab25.txt 2>&1
