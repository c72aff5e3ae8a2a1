O=gpurun_out/r29; mkdir -p $O
timeout 900 python -m pytest tests/test_fusions_gpu.py tests/test_varlen_gpu.py tests/test_parity_gpu.py -q -rf -x > $O/pytest_fast.log 2>&1; echo "rc=$?" >> $O/pytest_fast.log
timeout 900 bash tools/ab_fusions.sh 3 3 7 > $O/ab_fusions.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
