#!/bin/bash
# One GPU-box session of round-end evidence (outputs under gpurun_out/evidence/):
#   GPU tests (+ parity tables), smoke, the driver's bench command and the reference arm, a launch list with DRAM
#   bytes, ncu --set full captures of the dominant attention pass and the fused QKV GEMM exported as CSV on the box
#   (the .ncu-rep files stay in /tmp: gpurun copies back at most 64 MiB).
O=gpurun_out/evidence; mkdir -p $O; T=/tmp/ncu_evidence; mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
MGV_REPORT_DIR=$O/parity timeout 2400 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python tools/profile_step.py --steps 1 > $O/ncu_launch.log 2>&1
cap() {  # name, ncu filter args...
  n=$1; shift
  timeout 900 ncu --set full --clock-control none --import-source on "$@" -c 1 -o $T/$n -f python tools/profile_step.py --steps 0 > $O/ncu_$n.log 2>&1
  ncu -i $T/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>> $O/ncu_$n.log
  ncu -i $T/$n.ncu-rep --page details --csv > $O/$n.details.csv 2>> $O/ncu_$n.log
}
cap dkv -k regex:attn_bwd_dkv_v11 --launch-skip 1
cap qkv_fused --kernel-name-base demangled -k regex:EpiQKNormRope
echo all_done
