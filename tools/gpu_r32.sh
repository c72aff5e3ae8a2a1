O=gpurun_out/r32; mkdir -p $O
T=/tmp/ncu_r32; mkdir -p $T
cap() {  # name, ncu filter args...
  n=$1; shift
  timeout 900 ncu --set full --clock-control none --import-source on "$@" -c 1 -o $T/$n -f python tools/profile_step.py --steps 0 > $O/ncu_$n.log 2>&1; echo "rc=$?" >> $O/ncu_$n.log
  ncu -i $T/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>> $O/ncu_$n.log
  ncu -i $T/$n.ncu-rep --page details --csv > $O/$n.details.csv 2>> $O/ncu_$n.log
}
cap qkv_fused --kernel-name-base demangled -k regex:EpiQKNormRope
cap dkv -k regex:attn_bwd_dkv_v11 --launch-skip 1
cap storet --kernel-name-base demangled -k regex:EpiStoreT
ls -la $O
