O=gpurun_out/r31; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiQKNormRope -c 1 -o $O/qkv_fused -f python tools/profile_step.py --steps 0 > $O/ncu_qkv.log 2>&1; echo "rc=$?" >> $O/ncu_qkv.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dkv_v11 --launch-skip 1 -c 1 -o $O/dkv -f python tools/profile_step.py --steps 0 > $O/ncu_dkv.log 2>&1; echo "rc=$?" >> $O/ncu_dkv.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:EpiStoreT -c 1 -o $O/storet -f python tools/profile_step.py --steps 0 > $O/ncu_storet.log 2>&1; echo "rc=$?" >> $O/ncu_storet.log
