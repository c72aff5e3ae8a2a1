#!/bin/bash
# A/B whole-step kernel times of alternative library builds on the same box:
#   tools/ab_step.sh reps lib1 lib2 ...     (prints total + top kernels per run)
R=$1; shift
for r in $(seq 1 $R); do
  for lib in "$@"; do
    echo "== $lib"
    MGV_LIB_PATH=$lib python tools/profile_step.py --steps 3 --kernels 2>/dev/null | grep -E "total|attn|gemm" | head -12
  done
done
