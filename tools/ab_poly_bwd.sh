# A/B of the FMA-pipe exponential share in the attention backward (MGV_BWD_POLY = 0 / 4 / 2), alternating
for r in 1 2 3; do for P in 0 4 2; do
  echo "== POLY $P $(MGV_BWD_POLY=$P timeout 150 python tools/probe_attn.py 57600 bwd 5 kernels 2>&1 | grep -iE 'attn bwd|dkv|dq_v' | tr '\n' ' ' | cut -c1-330)"
done; done
