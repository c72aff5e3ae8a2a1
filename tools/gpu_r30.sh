O=gpurun_out/r30; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python tools/profile_step.py --steps 1 > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:EpiQKNormRope -c 1 -o $O/qkv_fused -f python tools/profile_step.py --steps 0 > $O/ncu_qkv.log 2>&1; echo "rc=$?" >> $O/ncu_qkv.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dkv_v11 -c 1 -o $O/dkv -f python tools/profile_step.py --steps 0 > $O/ncu_dkv.log 2>&1; echo "rc=$?" >> $O/ncu_dkv.log
