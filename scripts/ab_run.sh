#!/bin/bash
# per-worker pre-stage lanes: series tests (lanes forced and not), e2e probe at C3 T=3 with and without lanes
timeout 900 python -m pytest tests/test_gpu_series.py tests/test_gpu_preproc.py -x -q > gpurun_out/ab14_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab14_tests.log
for round in 1 2; do
  for l in 0 1; do RTN_PRE_LANES=$l timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-check 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lanes$l', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"; done
done > gpurun_out/ab14.txt 2>&1
