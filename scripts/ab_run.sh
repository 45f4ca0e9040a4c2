#!/bin/bash
# group tolerance mode (exact two-pass recurrence): channel and process-group tests, then the full suite
timeout 900 python -m pytest tests/test_gpu_channel.py tests/test_gpu_procgroup.py -x -q > gpurun_out/ab20_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab20_tests.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ab20_all.log 2>&1; echo "exit $?" >> gpurun_out/ab20_all.log
