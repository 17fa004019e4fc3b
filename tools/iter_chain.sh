# one iteration: chain parity tests, bench 5pc/3pc, ncu of a stage-3 chain pair
T=${1:-it}; O=gpurun_out/$T; mkdir -p $O
python -m pytest tests/test_gpu_batched.py tests/test_gpu_parity_batched.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
python bench.py --no-cpu-baseline --steps 5 > $O/bench5.json 2> $O/bench5.err; echo "bench5 rc=$?"
python bench.py --workload resnet152-3pc --no-cpu-baseline --steps 5 > $O/bench3.json 2> $O/bench3.err; echo "bench3 rc=$?"
python - <<'PY' $O
import json,sys
for f in ("bench5","bench3"):
    try:
        d=json.load(open(f"{sys.argv[1]}/{f}.json"))
        r=d["roofline_by_kernel"]
        print(f, d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"], "chain ms", r["chain"]["ms_per_step"], "gemm ms", r["gemm"]["ms_per_step"], "ok", d.get("outputs_match_plaintext"))
    except Exception as e: print(f, "ERR", e)
PY
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_chain --launch-skip 60 -c 2 -o $O/chain_full python tools/profile_step.py resnet152-5pc 32 > $O/ncu.log 2>&1; tail -1 $O/ncu.log
