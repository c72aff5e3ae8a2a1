O=gpurun_out/r4; mkdir -p $O
./tools/micro/mma_v11 > $O/mma_v11.log 2>&1
timeout 600 ncu --set full -k regex:dkv_v11 -c 1 --clock-control none --import-source on -f -o $O/dkv_v11 python tools/probe_attn.py 57600 bwd 1 > $O/ncu_v11.log 2>&1
timeout 600 ncu --set full -k regex:dq_v10 -c 1 --clock-control none --import-source on -f -o $O/dq_v10 python tools/probe_attn.py 57600 bwd 1 > $O/ncu_dq.log 2>&1
