#!/bin/bash
# One GPU-box session: GPU tests (+ parity tables), the reference CPU sweep on the host cores beside the bench,
# the bench itself, and compute-sanitizer on the smoke config.  Outputs under gpurun_out/r2/.
set -x
O=gpurun_out/r2; mkdir -p $O
nproc > $O/host.txt; free -g >> $O/host.txt; lscpu | head -20 >> $O/host.txt
MGV_REPORT_DIR=$O/parity timeout 3000 python -m pytest tests -m gpu -q -rf ${PYTEST_ARGS} > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
if [ -n "$SWEEP" ]; then (timeout 3000 python tools/cpu_sweep.py $O/cpu_sweep.json > $O/cpu_sweep.log 2>&1) & SW=$!; fi
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
if [ -n "$SANITIZE" ]; then
  timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/memcheck.log 2>&1; echo "rc=$?" >> $O/memcheck.log
  timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/synccheck.log 2>&1; echo "rc=$?" >> $O/synccheck.log
fi
if [ -n "$SW" ]; then wait $SW; fi
echo done
