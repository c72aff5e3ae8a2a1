#!/bin/bash
# SM clock / power while a probe runs:  tools/clock_probe.sh <label> <command...>
label=$1; shift
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 20 > /tmp/clk_$$.csv &
pid=$!
sleep 0.3
"$@" | sed "s/^/$label /"
kill $pid
awk -F, -v l="$label" '$2+0 > 400 {n++; c+=$1; p+=$2} END {if (n) printf("%s: %d samples under load, SM %.0f MHz, %.0f W\n", l, n, c/n, p/n)}' /tmp/clk_$$.csv
