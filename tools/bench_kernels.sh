#!/bin/bash
# quick: gpu nn/network tests + bench with per-kernel table
mkdir -p gpurun_out
timeout 600 python -m pytest --timeout 300 -x -q tests/test_gpu_nn.py tests/test_gpu_networks.py > gpurun_out/pytest_nn.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nn.log
tail -n 3 gpurun_out/pytest_nn.log
timeout 900 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
l = json.loads(open('gpurun_out/bench.log').readline())
print("value", l['value'], "ms/step", l['ms_per_step'], "e2e", (l.get('e2e') or {}).get('value'))
for r in l['roofline_kernels']:
    print(f"{r['kernel']:24s} n={r['launches']:5d} ms={r['ms_total']:8.2f} share={r['share_of_step_time']:.3f} ach={r['achieved']:.0f} {r['unit']} frac={r['frac']:.3f}")
PY
