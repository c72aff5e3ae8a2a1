O=gpurun_out/r15; mkdir -p $O
python tools/profile_step.py --steps 1 > $O/plain.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv python tools/profile_step.py --steps 1 > $O/ncu_list.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_dkv_v11|attn_bwd_dq_v10|attn_fwd_tc" -c 6 -f -o $O/attn_full python tools/profile_step.py --steps 0 > $O/ncu_full.log 2>&1
