O=gpurun_out/r22; mkdir -p $O
MGV_ATTN_FWD1=1 timeout 600 python -m pytest tests/test_attn_gpu.py tests/test_varlen_gpu.py -q -x > $O/tests_fwd1.log 2>&1; echo "rc=$?" >> $O/tests_fwd1.log
for r in 1 2 3; do for V in 0 1; do echo "== FWD1 $V $(MGV_ATTN_FWD1=$V timeout 150 python tools/probe_attn.py 57600 fwd 10 kernels 2>&1 | grep -iE 'attn fwd|attn_fwd' | tr '\n' ' ' | cut -c1-220)"; done; done > $O/ab_fwd.log
