O=gpurun_out/r5; mkdir -p $O
timeout 900 python -m pytest tests/test_attn_gpu.py -q -x > $O/attn_tests.log 2>&1; echo "rc=$?" >> $O/attn_tests.log
timeout 900 bash tools/ab_dkv.sh > $O/ab_dkv.log 2>&1
timeout 600 ncu --set full -k regex:dkv_v11 -c 1 --clock-control none --import-source on -f -o $O/dkv_v11 python tools/probe_attn.py 57600 bwd 1 > $O/ncu_v11.log 2>&1
