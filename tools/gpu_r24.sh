O=gpurun_out/r24; mkdir -p $O
timeout 900 python -m pytest tests/test_qkv_fused_gpu.py tests/test_parity_gpu.py tests/test_tp_gpu.py tests/test_varlen_gpu.py -q -rf -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-extra --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-extra --no-cpu-baseline > $O/ncu.log 2>&1; echo "rc=$?" >> $O/ncu.log
