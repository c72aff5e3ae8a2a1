O=gpurun_out/r34; mkdir -p $O
timeout 1500 bash tools/ab_fusions_full.sh 4 6 7 > $O/ab_full.log 2>&1
