O=gpurun_out/r28; mkdir -p $O
timeout 900 python -m pytest tests/test_tp_gpu.py tests/test_fusions_gpu.py -q -rf -s > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python tools/tp_exchange.py --sizes 2 8 --steps 3 > $O/tp_exchange_f32.log 2>&1; echo "rc=$?" >> $O/tp_exchange_f32.log
MGV_TP_PAYLOAD=bf16 timeout 600 python tools/tp_exchange.py --sizes 2 8 --steps 3 > $O/tp_exchange_bf16.log 2>&1; echo "rc=$?" >> $O/tp_exchange_bf16.log
