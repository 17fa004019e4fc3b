# A/B a list of env settings on the bench: bash tools/ab_env.sh TAG WORKLOAD "ENV1" "ENV2" ...
T=$1; W=$2; shift 2; O=gpurun_out/$T; mkdir -p $O
for e in "$@"; do
  n=$(echo "$e" | tr ' =/' '___')
  env $e python bench.py --workload $W --no-cpu-baseline --steps 5 > $O/$n.json 2> $O/$n.err
  python -c "
import json,sys
d=json.load(open('$O/$n.json')); r=d['roofline_by_kernel']
print('$e', d['value'], 'ms', d['ms_per_step'], 'chain', r['chain']['ms_per_step'], 'gemm', r['gemm']['ms_per_step'], 'ok', d.get('outputs_match_plaintext'))" 2>&1 | tail -1
done
