O=gpurun_out/r10; mkdir -p $O
timeout 900 python -m pytest tests/test_attn_gpu.py -q -x > $O/attn_tests.log 2>&1; echo "rc=$?" >> $O/attn_tests.log
timeout 900 bash tools/ab_dkv.sh > $O/ab_dkv.log 2>&1
python tools/trace_dkv11.py 57600 > $O/trace.log 2>&1
