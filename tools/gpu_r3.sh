O=gpurun_out/r3; mkdir -p $O
(timeout 3000 python tools/cpu_sweep.py $O/cpu_sweep.json > $O/cpu_sweep.log 2>&1) & SW=$!
timeout 900 python -m pytest tests/test_attn_gpu.py -q -x > $O/attn_tests.log 2>&1; echo "rc=$?" >> $O/attn_tests.log
timeout 900 bash tools/ab_dkv.sh > $O/ab_dkv.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py -q -x > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extra > $O/bench.json 2> $O/bench.err
wait $SW
