#!/bin/bash
# A/B of the ws A^H A unit ranges (option rank_vh) + the A^H A parity tests
mkdir -p gpurun_out
SH="320 368 15 8 512 512 32 4 256 256 8 16"
: > gpurun_out/vh.log
for rep in 1 2; do
for vh in 0 9 ${VHS}; do
  echo "== rank_vh=$vh" >> gpurun_out/vh.log
  timeout 300 python tools/sense_bench.py $SH --iters 20 --opt rank_vh=$vh >> gpurun_out/vh.log 2>&1
done
done
timeout 900 python -m pytest -q -x tests/test_gpu_sense_rank.py tests/test_gpu_sense.py tests/test_gpu_golden.py > gpurun_out/vh_tests.log 2>&1; tail -2 gpurun_out/vh_tests.log
python - <<'PY'
import json
for line in open("gpurun_out/vh.log"):
    if line.startswith("=="): print(line.strip()); continue
    if line.startswith("{"):
        d = json.loads(line)
        print(f'  {d["X"]}x{d["Y"]}x{d["coils"]}x{d["B"]}: cg launch {d.get("sense_normal_y_cg_us",0):.1f} us ({d.get("sense_normal_y_cg_gbs",0):.0f} GB/s)  apply {d["apply_us"]:.1f} us  cg10 {d["cg10_ms"]*1e3:.0f} us')
PY
