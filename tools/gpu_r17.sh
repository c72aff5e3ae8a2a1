O=gpurun_out/r18; mkdir -p $O
timeout 600 python -m pytest tests/test_varlen_gpu.py tests/test_attn_gpu.py -q -x > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for r in 1 2 3; do timeout 150 python tools/probe_attn.py 57600 bwd 5 kernels 2>&1 | grep -iE 'attn bwd|dkv|dq_v' | tr '\n' ' ' | cut -c1-330; echo; done > $O/probe.log
