#!/bin/bash
# Round measurement: default bench line, every BASELINE config, C4 as configured (8 frames
# in flight, t-k schedule), the N>1 headline path on this GPU, the launch list and one
# ncu --set full summary of the C3 kernels. TAG names the outputs.
TAG=${TAG:-r02v5}; O=gpurun_out; mkdir -p $O
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
for c in c1 c2 c4 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-check 2>>$O/${TAG}_configs.err; done > $O/${TAG}_configs.jsonl
timeout 600 python bench.py --config c4 --T 8 --sched 5,8 --no-cpu-baseline 2>>$O/${TAG}_configs.err > $O/${TAG}_c4_t8.json
timeout 600 python scripts/decomp_bench_check.py c3 2 > $O/${TAG}_single_series_2dev.json 2>&1
RTN_PROFILE_STEP=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --T 3 --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-check > $O/${TAG}_launches.log 2>&1
REPS=2 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o $O/${TAG}_full -f python scripts/prof_kernels.py c3 colA rows1 colsT rows2 colsW cr_fused crA > $O/${TAG}_full.log 2>&1
python profiles/summarize.py full $O/${TAG}_full.ncu-rep > $O/${TAG}_full_summary.json 2>&1
ncu -i $O/${TAG}_full.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/${TAG}_full_raw.csv.gz
rm -f $O/${TAG}_full.ncu-rep
REPS=50 timeout 300 python scripts/prof_kernels.py c3 colA rows1 colsT rows2 colsW cr_fused crA apply > $O/${TAG}_isolated.txt 2>&1
