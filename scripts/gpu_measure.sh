#!/bin/bash
# One measurement pass on a B200 box (run under gpurun): GPU tests, the default bench line,
# the launch list of the timed step and one ncu --set full capture of the hot kernels.
# TAG names the outputs (gpurun_out/<TAG>_*).
TAG=${TAG:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/${TAG}_pytest_gpu.log
fi
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
RTN_PROFILE_STEP=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --T 3 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-check > $O/${TAG}_launches.log 2>&1
REPS=2 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o $O/${TAG}_full -f python scripts/prof_kernels.py c3 colA rows1 colsT rows2 colsW cr_fused crA > $O/${TAG}_full.log 2>&1
REPS=50 timeout 300 python scripts/prof_kernels.py c3 colA rows1 colsT rows2 colsW cr_fused crA apply > $O/${TAG}_isolated.txt 2>&1
# summarise on the box; the .ncu-rep itself is too large to come back (gpurun_out <= 64 MiB)
python profiles/summarize.py full $O/${TAG}_full.ncu-rep > $O/${TAG}_full_summary.json 2>&1
ncu -i $O/${TAG}_full.ncu-rep --page raw --csv > $O/${TAG}_full_raw.csv 2>/dev/null
ncu -i $O/${TAG}_full.ncu-rep --page source --csv --kernel-name regex:colsW > $O/${TAG}_src_colsW.csv 2>/dev/null
gzip -f $O/${TAG}_full_raw.csv $O/${TAG}_src_colsW.csv
rm -f $O/${TAG}_full.ncu-rep
ls -la $O
