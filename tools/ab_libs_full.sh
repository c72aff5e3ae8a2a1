#!/bin/bash
# Full per-kernel tables of alternating runs of alternative library builds: tools/ab_libs_full.sh reps lib...
R=$1; shift
for r in $(seq 1 $R); do
  for lib in "$@"; do
    echo "== lib $lib"
    MGV_LIB_PATH=$lib TOPK=200 python tools/profile_step.py --steps 4 --kernels 2>/dev/null | grep -vE "^step [0-3]:"
  done
done
