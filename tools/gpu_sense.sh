#!/bin/bash
# SENSE-only GPU pass: sense parity tests + micro-bench (+ optional ncu of k_normal)
# SWEEP="opts1;opts2" runs the micro-bench once per option set (space-separated key=value)
mkdir -p gpurun_out
timeout 600 python -m pytest --timeout 120 tests/test_gpu_sense_rank.py tests/test_gpu_sense.py tests/test_gpu_golden.py -x -q > gpurun_out/pytest_sense.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sense.log
: > gpurun_out/sense_bench.log
IFS=';' read -ra SETS <<< "${SWEEP:-}"
[ ${#SETS[@]} -eq 0 ] && SETS=("")
for set in "${SETS[@]}"; do
  args=""
  for kv in $set; do args="$args --opt $kv"; done
  echo "== opts: $set" >> gpurun_out/sense_bench.log
  timeout 300 python tools/sense_bench.py 320 368 15 8 640 368 15 4 256 256 8 16 512 512 32 4 $args >> gpurun_out/sense_bench.log 2>&1
done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_normal -s 6 -c 2 \
   -o gpurun_out/prof_sense -f python tools/sense_bench.py 320 368 15 8 --iters 4 > gpurun_out/ncu_sense.log 2>&1
fi
tail -15 gpurun_out/pytest_sense.log; cat gpurun_out/sense_bench.log
