O=gpurun_out/r27; mkdir -p $O
timeout 1500 bash tools/ab_bwd.sh paper_2510_17519_b200/libmugv_b200.so ab_libs/dkvx1/libmugv_b200.so ab_libs/dkvx2/libmugv_b200.so ab_libs/dkvx4/libmugv_b200.so ab_libs/dkvx7/libmugv_b200.so > $O/ab_dkvx.log 2>&1
