O=gpurun_out/r33; mkdir -p $O
timeout 900 python -m pytest tests/test_fusions_gpu.py tests/test_parity_gpu.py tests/test_parity_golden_gpu.py -q -rf -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 bash tools/ab_fusions.sh 3 6 7 > $O/ab_fusions.log 2>&1
