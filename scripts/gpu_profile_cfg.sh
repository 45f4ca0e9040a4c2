#!/bin/bash
# isolated timings + one ncu --set full capture (summarised on the box) of one config's
# pass kernels: CFG=c5 TAG=c5_v1 bash scripts/gpu_profile_cfg.sh
CFG=${CFG:-c5}; TAG=${TAG:-${CFG}}; O=gpurun_out; mkdir -p $O
KER=${KER:-"colA rows1 colsT rows2 colsW cr_fused crA"}
REPS=30 timeout 300 python scripts/prof_kernels.py $CFG $KER apply > $O/${TAG}_isolated.txt 2>&1
REPS=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -o $O/${TAG}_full -f python scripts/prof_kernels.py $CFG $KER > $O/${TAG}_full.log 2>&1
python profiles/summarize.py full $O/${TAG}_full.ncu-rep > $O/${TAG}_full_summary.json 2>&1
ncu -i $O/${TAG}_full.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/${TAG}_full_raw.csv.gz
if [ -n "$SRC" ]; then ncu -i $O/${TAG}_full.ncu-rep --page source --csv --kernel-name regex:$SRC 2>/dev/null | gzip > $O/${TAG}_src.csv.gz; fi
rm -f $O/${TAG}_full.ncu-rep
