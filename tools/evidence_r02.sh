# Round-2 evidence on one B200: int8 peak probe, GPU tests, bench lines (ResNet-152 5PC/3PC, GEMM sweep, LeNet-28) and the reference arm.  Usage: bash tools/evidence_r02.sh TAG
O=gpurun_out/${1:-r2}; mkdir -p $O
python tools/int8_peak.py $O/int8_peak.json
python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
python bench.py > $O/bench_resnet152.json 2> $O/bench_resnet152.err; echo "bench rc=$?"
python bench.py --workload resnet152-3pc --no-cpu-baseline > $O/bench_resnet152_3pc.json 2> $O/bench_resnet152_3pc.err
python bench.py --workload gemm-sweep > $O/bench_gemm.json 2> $O/bench_gemm.err; echo "gemm rc=$?"
python bench.py --workload lenet28-3pc > $O/bench_lenet28.json 2> $O/bench_lenet28.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
for f in $O/*.err; do echo "== $f"; tail -n 3 $f; done
