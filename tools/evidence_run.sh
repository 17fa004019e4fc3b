# Round evidence on one B200: GPU tests, smoke, bench lines for every workload (+ the reference
# arm), the per-kernel launch list and DRAM traffic of one step.  Usage: bash tools/evidence_run.sh TAG
set -x
T=${1:-vX}
O=gpurun_out/$T
mkdir -p $O
python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python bench.py > $O/bench_resnet152.json 2> $O/bench_resnet152.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for w in resnet50-3pc resnet18-cifar-3pc lenet28-3pc gemm-sweep; do
  python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/launches.csv python tools/profile_step.py > $O/ncu1.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/traffic.csv python tools/profile_step.py > $O/ncu2.log 2>&1
