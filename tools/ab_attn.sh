#!/bin/bash
# A/B the attention kernels of alternative builds on the same box: tools/ab_attn.sh N reps lib1 lib2 ...
N=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for lib in "$@"; do
    echo "== $lib"
    MGV_LIB_PATH=$lib python tools/probe_attn.py $N both 3 kernels 2>/dev/null | grep -E "attn_(fwd|bwd)_|dq|dkv"
  done
done
