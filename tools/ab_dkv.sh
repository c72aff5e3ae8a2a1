# A/B of the dK/dV pass (v11 default vs v8 via MGV_DKV_V8=1), alternating on one box, 57,600 tokens x 24 x 144
for r in 1 2 3; do
  echo "== v11 $(timeout 150 python tools/probe_attn.py 57600 bwd 5 kernels 2>&1 | grep -iE 'attn bwd|dkv|dq_v' | tr '\n' ' ')"

done
