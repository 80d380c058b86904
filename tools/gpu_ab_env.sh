#!/bin/bash
# A/B of a bench workload under an MDNN_* option env var: AB_VAR (e.g. MDNN_RBF_PAIR),
# AB_VALS (e.g. "1 0"), WL (workload); prints value + per-tag ms_total
mkdir -p gpurun_out
: > gpurun_out/ab_env.log
for rep in 1 2; do for v in $AB_VALS; do
  echo "== $AB_VAR=$v" >> gpurun_out/ab_env.log
  env $AB_VAR=$v timeout 600 python bench.py --workload $WL --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(' value', round(d['value'],2))
for k in d['roofline_kernels'][:8]: print('  ', k['kernel'], round(k['frac'],3), round(k['ms_total'],3))
" >> gpurun_out/ab_env.log
done; done
cat gpurun_out/ab_env.log
