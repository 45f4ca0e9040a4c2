#!/bin/bash
# Build library variants into build_var/ (here, on the CPU) for same-box A/B runs:
#   scripts/build_variants.sh name "<extra nvcc flags>" [name "<flags>" ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p build_var
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  RTN_NVCC_EXTRA="$flags" python -c "
import sys; sys.path.insert(0, 'paper_1701_08361_b200')
import build; build.build(force=True, out='build_var/lib_$name.so')" > /dev/null
  echo "built build_var/lib_$name.so ($flags)"
done
