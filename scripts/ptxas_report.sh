#!/bin/bash
# registers and spills per pass kernel of one instantiation unit: scripts/ptxas_report.sh inst3.cu [extra nvcc flags]
cd "$(dirname "$0")/../paper_1701_08361_b200/csrc"
src=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -Xptxas=-v "$@" -c $src -o /tmp/ptxas_report.o 2>&1 | python3 -c "
import sys,re,subprocess
name=None;st=None
for line in sys.stdin:
    m=re.search(r\"Compiling entry function '(\S+)'\",line)
    if m: name=subprocess.run(['c++filt',m.group(1)],capture_output=True,text=True).stdout.split('(')[0].replace('rtnb::','').replace('void ',''); continue
    m=re.search(r'(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads',line)
    if m and name: st=m.groups()
    m=re.search(r'Used (\d+) registers',line)
    if m and name and 'k_' in name: print(name, 'regs',m.group(1),'stack/spill-st/spill-ld',st); name=None
"
