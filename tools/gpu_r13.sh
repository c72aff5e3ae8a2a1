O=gpurun_out/r14; mkdir -p $O
timeout 1200 python -m pytest tests/test_varlen_gpu.py tests/test_tp_gpu.py tests/test_attn_gpu.py -q -rf -x > $O/varlen.log 2>&1; echo "rc=$?" >> $O/varlen.log
timeout 3000 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
