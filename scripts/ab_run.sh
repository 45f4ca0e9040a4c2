#!/bin/bash
# same-box A/B: base (previous commit) vs the working tree; then the whole-step DRAM ranges
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_configs.py -x -q -k "384 or c5 or 24 or c2 or 320" > gpurun_out/ab9_tests.log 2>&1; echo "exit $?" >> gpurun_out/ab9_tests.log
for round in 1 2; do
  for lib in base new; do
    if [ $lib = new ]; then export RTN_LIB=$PWD/paper_1701_08361_b200/librtnlinv_b200.so; else export RTN_LIB=$PWD/build_var/lib_$lib.so; fi
    for c in c5; do timeout 120 python scripts/decomp_probe.py $c 2x1 1x1 | sed "s/^/$lib $c /"; done
    REPS=30 timeout 120 python scripts/prof_kernels.py c5 rows1 rows2 | sed "s/^/$lib /"
  done
done > gpurun_out/ab9.txt 2>&1
unset RTN_LIB
for a in "c3 3 8" "c5 2 4"; do
  set -- $a
  timeout 900 ncu --replay-mode app-range --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --csv python scripts/step_range.py $1 $2 $3 > gpurun_out/range_$1.csv 2>&1
done
