O=gpurun_out/r12; mkdir -p $O
timeout 1200 python -m pytest tests/test_tp_gpu.py tests/test_adamw_gpu.py tests/test_parity_gpu.py -q -rf > $O/tp.log 2>&1; echo "rc=$?" >> $O/tp.log
timeout 3000 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
