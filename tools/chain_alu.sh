# Chain ALU calibration (bench.py CHAIN_ALU) for the ResNet-152 workloads: bash tools/chain_alu.sh TAG
O=gpurun_out/${1:-alu}; mkdir -p $O
for W in resnet152-5pc resnet152-3pc; do
  ncu --metrics smsp__thread_inst_executed.sum,sm__pipe_fmaheavy_cycles_active.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg \
      --clock-control none --profile-from-start off -k regex:k_chain --csv --log-file $O/$W.csv \
      python tools/profile_step.py $W 32 > $O/$W.log 2>&1
  python tools/chain_alu.py $W 32 $O/$W.csv
done
