O=gpurun_out/r39; mkdir -p $O
for r in 1 2 3; do for lib in paper_2510_17519_b200/libmugv_b200.so ab_libs/dqx2/libmugv_b200.so ab_libs/dqp4/libmugv_b200.so ab_libs/dqp3/libmugv_b200.so; do
  echo "== $lib"; MGV_LIB_PATH=$lib timeout 150 python tools/probe_attn.py 57600 bwd 5 kernels 2>&1 | grep -E "attn_bwd_d"
done; done > $O/ab_dq.log 2>&1
