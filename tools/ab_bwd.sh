# A/B of two builds of the attention backward, alternating on one box: tools/ab_bwd.sh libA libB
for r in 1 2 3 4; do for lib in "$@"; do echo "== $lib"; MGV_LIB_PATH=$lib timeout 150 python tools/probe_attn.py 57600 bwd 5 kernels 2>&1 | grep -iE "attn_bwd|dq|dkv"; done; done
