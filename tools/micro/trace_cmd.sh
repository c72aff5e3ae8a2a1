python tools/trace_attn.py | tail -4
(nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader -lms 100 > gpurun_out/smi2.csv &)
sleep 0.5
python tools/probe_attn.py 57600 bwd 4 kernels | grep -E "dq|dkv"
sleep 0.3
awk -F, '$2+0>300' gpurun_out/smi2.csv | sort | uniq -c | sort -rn | head -8
