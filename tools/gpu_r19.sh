O=gpurun_out/r19; mkdir -p $O
MGV_DKV_CW=4 timeout 600 python -m pytest tests/test_attn_gpu.py tests/test_varlen_gpu.py -q -x > $O/tests_cw4.log 2>&1; echo "rc=$?" >> $O/tests_cw4.log
for r in 1 2 3; do for C in 2 4; do echo "== CW $C $(MGV_DKV_CW=$C timeout 150 python tools/probe_attn.py 57600 bwd 5 kernels 2>&1 | grep -iE 'attn bwd|dkv' | tr '\n' ' ' | cut -c1-200)"; done; done > $O/ab_cw.log
