O=gpurun_out/r36; mkdir -p $O
timeout 1500 python -m pytest tests/test_parity_golden_gpu.py -q -rf -s -k tp_step > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
