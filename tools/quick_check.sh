# quick GPU check: GEMM/engine parity tests, bench line, per-kernel launch list
mkdir -p gpurun_out/gq
python -m pytest tests/test_gpu_gemm_tc.py tests/test_gpu_batched.py -q -x 2>&1 | tail -3
python bench.py --no-cpu-baseline > gpurun_out/gq/bench.json 2> gpurun_out/gq/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/gq/launches.csv python tools/profile_step.py > gpurun_out/gq/ncu.log 2>&1
