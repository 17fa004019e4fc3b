set -x
mkdir -p gpurun_out/v9
python -m pytest tests -m gpu -q -x > gpurun_out/v9/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/v9/pytest_gpu.log
python bench.py > gpurun_out/v9/bench_resnet152.json 2> gpurun_out/v9/bench_resnet152.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v9/bench_ref.json 2> gpurun_out/v9/bench_ref.err
for w in resnet50-3pc resnet18-cifar-3pc lenet28-3pc; do python bench.py --workload $w > gpurun_out/v9/bench_$w.json 2> gpurun_out/v9/bench_$w.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/v9/launches.csv python tools/profile_step.py > gpurun_out/v9/ncu1.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/v9/traffic.csv python tools/profile_step.py > gpurun_out/v9/ncu2.log 2>&1
