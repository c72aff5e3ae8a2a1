O=gpurun_out/r37; mkdir -p $O
timeout 1500 bash tools/ab_libs_full.sh 3 paper_2510_17519_b200/libmugv_b200.so ab_libs/rpc32/libmugv_b200.so > $O/ab_rpc.log 2>&1
