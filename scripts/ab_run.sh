#!/bin/bash
# sanity after the enqueue-mode guard: channel, series, config tests and the default bench line
timeout 1500 python -m pytest tests/test_gpu_channel.py tests/test_gpu_series.py tests/test_gpu_configs.py tests/test_gpu_ops.py -x -q > gpurun_out/ab16_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab16_tests.log
timeout 600 python bench.py > gpurun_out/ab16_bench.json 2> gpurun_out/ab16_bench.err
