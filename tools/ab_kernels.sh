# Per-kernel ncu time of one profiled step for several library builds / env settings:
#   bash tools/ab_kernels.sh TAG WORKLOAD BATCH "ENV1" "ENV2" ...   (ENV e.g. "SSN_LIB=exp/lib_head.so")
T=$1; W=$2; B=$3; shift 3; O=gpurun_out/$T; mkdir -p $O
for e in "$@"; do
  n=$(echo "$e" | tr ' =/' '___')
  env $e ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file $O/$n.csv python tools/profile_step.py $W $B > $O/$n.log 2>&1
  echo "== $e"; python tools/kernel_table.py $O/$n.csv 2>/dev/null | grep -E "chain|gemm|TOTAL"
done
