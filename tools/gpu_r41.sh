O=gpurun_out/r41; mkdir -p $O
timeout 900 python -m pytest tests/test_recompute_gpu.py tests/test_tp_gpu.py tests/test_varlen_gpu.py tests/test_parity_gpu.py -q -rf -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 1200 python tools/stack_train.py --depth 24 --steps 3 --warmup 2 --grid 16 45 80 --recompute > $O/stack_d24_57k_rc.log 2>&1; echo "rc=$?" >> $O/stack_d24_57k_rc.log
cp gpurun_out/stack_train_*.json $O/ 2>/dev/null
