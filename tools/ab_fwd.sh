# A/B of two builds of the attention forward, alternating on one box: tools/ab_fwd.sh libA libB
for r in 1 2 3 4 5; do for lib in "$@"; do echo "== $lib $(MGV_LIB_PATH=$lib timeout 120 python tools/probe_attn.py 57600 fwd 10 2>&1 | grep -iE 'attn fwd')"; done; done
