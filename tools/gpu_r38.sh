O=gpurun_out/r38; mkdir -p $O
timeout 600 python -m pytest tests/test_attn_gpu.py -q -rf -x > $O/pytest_attn.log 2>&1; echo "rc=$?" >> $O/pytest_attn.log
for r in 1 2 3; do for lib in ab_libs/fpoly0/libmugv_b200.so paper_2510_17519_b200/libmugv_b200.so ab_libs/fpoly3/libmugv_b200.so ab_libs/fpoly8/libmugv_b200.so; do
  echo "== $lib"; MGV_LIB_PATH=$lib timeout 150 python tools/probe_attn.py 57600 fwd 10 2>&1 | grep -E "attn fwd"
done; done > $O/ab_fpoly.log 2>&1
timeout 1500 bash tools/ab_libs_full.sh 2 ab_libs/fpoly0/libmugv_b200.so paper_2510_17519_b200/libmugv_b200.so > $O/ab_step.log 2>&1
