#!/bin/bash
# A/B of the forward fusions on one box: alternating runs with mgv_dev_set_fusions masks (0 = unfused)
#   tools/ab_fusions.sh reps mask1 mask2 ...
R=$1; shift
for r in $(seq 1 $R); do
  for m in "$@"; do
    echo "== fusions $m"
    python tools/profile_step.py --steps 3 --kernels --fusions $m 2>/dev/null | grep -E "^step 3|total|EpiQK|EpiStore|qk_norm|rms_fwd|postnorm|transpose" | head -14
  done
done
