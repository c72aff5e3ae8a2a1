O=gpurun_out/r26; mkdir -p $O
timeout 1200 python -m pytest tests/test_fusions_gpu.py tests/test_parity_gpu.py tests/test_tp_gpu.py -q -rf -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 bash tools/ab_fusions.sh 3 0 3 > $O/ab_fusions.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --steps 3 --warmup 3 --no-extra --no-cpu-baseline --depth 12 --grid 7 60 104 > $O/bench_d12.json 2> $O/bench_d12.err; echo "rc=$?" >> $O/bench_d12.err
