O=gpurun_out/r21; mkdir -p $O
timeout 1200 python -m pytest tests/test_dp_gpu.py tests/test_varlen_gpu.py tests/test_shim_gpu.py tests/test_tp_gpu.py -q -rf > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
