# A/B of one kernel's ncu duration between two builds (serialized launches, same box): tools/ab_kernel.sh REGEX libA libB
RX=$1; shift
for r in 1 2; do for lib in "$@"; do
  MGV_LIB_PATH=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$RX --csv python bench.py --steps 1 --warmup 0 --no-extra --no-cpu-baseline 2>/dev/null | grep -E "gpu__time_duration" | awk -F'","' -v L=$lib '{gsub(/"/,"",$NF); s+=$NF; n++} END {print L, n, "launches, mean", s/n, "ns"}'
done; done
