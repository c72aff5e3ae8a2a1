O=gpurun_out/r11; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
