# A/B of the softmax exponential split in the attention forward (MGV_ATTN_POLY), alternating on one box
for r in 1 2 3 4 5; do for P in 0 4; do echo "== POLY $P $(MGV_ATTN_POLY=$P timeout 120 python tools/probe_attn.py 57600 fwd 10 2>&1 | grep -iE 'attn fwd')"; done; done
