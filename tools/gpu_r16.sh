O=gpurun_out/r16; mkdir -p $O
for P in 4 2; do MGV_BWD_POLY=$P timeout 600 python -m pytest tests/test_attn_gpu.py -q -x 2>&1 | tail -1 > $O/attn_tests_p$P.log; done
timeout 1200 bash tools/ab_poly_bwd.sh > $O/ab_poly.log 2>&1
