O=gpurun_out/r22; mkdir -p $O
timeout 1200 python tools/stack_train.py --depth 24 > $O/stack_train.log 2>&1; echo "rc=$?" >> $O/stack_train.log
timeout 900 python tools/stack_fwd.py 2 > $O/stack_fwd.log 2>&1; echo "rc=$?" >> $O/stack_fwd.log
timeout 600 python tools/tp_exchange.py --sizes 2 8 --steps 3 > $O/tp_exchange.log 2>&1; echo "rc=$?" >> $O/tp_exchange.log
timeout 3000 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
