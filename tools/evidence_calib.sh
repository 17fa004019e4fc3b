# Calibration + profiles for the bench's roofline fields: chain ALU / heavy-pipe per element
# (bench.py CHAIN_ALU / CHAIN_HEAVY), DRAM traffic per kernel class (traffic.json), the ncu
# launch list of one step and an ncu --set full capture of the chain kernels.
# Usage: bash tools/evidence_calib.sh TAG
O=gpurun_out/${1:-calib}; mkdir -p $O
bash tools/chain_alu.sh ${1:-calib}/alu
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    --profile-from-start off --csv --log-file $O/traffic.csv python tools/profile_step.py resnet152-5pc > $O/traffic.log 2>&1
python tools/traffic.py $O/traffic.csv > $O/traffic.json; echo "traffic rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file $O/launches.csv python tools/profile_step.py resnet152-5pc > $O/launches.log 2>&1
python tools/kernel_table.py $O/launches.csv > $O/kernel_table.txt; head -12 $O/kernel_table.txt
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_chain --launch-skip 60 -c 2 \
    -o $O/chain_full python tools/profile_step.py resnet152-5pc 32 > $O/ncu_full.log 2>&1; tail -1 $O/ncu_full.log
