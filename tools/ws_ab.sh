#!/bin/bash
# A/B timing of the A^H A kernels: default build, optional alternative builds
# (MDNN_B200_LIB), and the previous k_normal_rank (sense_ws=0)
mkdir -p gpurun_out
SH="320 368 15 8 512 512 32 4 256 256 8 16"
: > gpurun_out/ab.log
echo "== default" >> gpurun_out/ab.log
timeout 300 python tools/sense_bench.py $SH --iters 20 >> gpurun_out/ab.log 2>&1
for lib in $ALT_LIBS; do
  echo "== $lib" >> gpurun_out/ab.log
  MDNN_B200_LIB=$lib timeout 300 python tools/sense_bench.py $SH --iters 20 >> gpurun_out/ab.log 2>&1
done
echo "== sense_ws=0" >> gpurun_out/ab.log
timeout 300 python tools/sense_bench.py $SH --iters 20 --opt sense_ws=0 ${ALT_OPT} >> gpurun_out/ab.log 2>&1
if [ -n "$TESTS" ]; then timeout 600 python -m pytest -q -x tests/test_gpu_sense_rank.py tests/test_gpu_sense.py tests/test_gpu_golden.py > gpurun_out/ab_tests.log 2>&1; tail -2 gpurun_out/ab_tests.log; fi
python - <<'PY'
import json
for line in open("gpurun_out/ab.log"):
    if line.startswith("=="): print(line.strip()); continue
    if line.startswith("{"):
        d = json.loads(line)
        print(f'  {d["X"]}x{d["Y"]}x{d["coils"]}x{d["B"]}: cg launch {d.get("sense_normal_y_cg_us",0):.1f} us ({d.get("sense_normal_y_cg_gbs",0):.0f} GB/s)  apply {d["apply_us"]:.1f} us  cg10 {d["cg10_ms"]*1e3:.0f} us')
PY
