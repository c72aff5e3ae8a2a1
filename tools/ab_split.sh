# A/B of the TMEM-load overlap in the attention backward: committed build vs early dP load in dQ (B) vs B + split
# S^T load in dK/dV after 16 / 32 columns (S16 / S32); 57,600 tokens x 24 x 144, alternating on one box
L=paper_2510_17519_b200
for lib in B S16 S32; do
  MGV_LIB_PATH=$L/libmugv_b200_$lib.so timeout 600 python -m pytest -q -x tests/test_attn_gpu.py tests/test_varlen_gpu.py 2>&1 | tail -1 | sed "s/^/[$lib tests] /"
done
for r in 1 2 3; do for lib in A B S16 S32; do
  P=$L/libmugv_b200_$lib.so; [ $lib = A ] && P=$L/libmugv_b200.so
  echo "== $lib $(MGV_LIB_PATH=$P timeout 150 python tools/probe_attn.py 57600 bwd 5 kernels 2>&1 | grep -iE 'attn bwd|dkv|dq_v' | tr '\n' ' ' | cut -c1-330)"
done; done
