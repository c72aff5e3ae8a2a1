#!/bin/bash
# Full per-kernel tables of alternating runs with mgv_dev_set_fusions masks: tools/ab_fusions_full.sh reps mask...
R=$1; shift
for r in $(seq 1 $R); do
  for m in "$@"; do
    echo "== fusions $m"
    TOPK=200 python tools/profile_step.py --steps 4 --kernels --fusions $m 2>/dev/null | grep -vE "^step [0-3]:"
  done
done
