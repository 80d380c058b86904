#!/bin/bash
# Profiling pass on the GPU box: SENSE micro-bench + ncu --set full of the
# named kernels.  KREGEX: kernel regex for the bench capture (optional).
mkdir -p gpurun_out
timeout 300 python tools/sense_bench.py 320 368 15 8 256 256 8 16 512 512 32 4 > gpurun_out/sense_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_normal -s 6 -c 2 \
   -o gpurun_out/prof_sense -f python tools/sense_bench.py 320 368 15 8 --iters 4 > gpurun_out/ncu_sense.log 2>&1
if [ -n "$KREGEX" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$KREGEX" -c ${KCOUNT:-6} \
   -o gpurun_out/prof_bench -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
fi
tail -2 gpurun_out/ncu_sense.log gpurun_out/ncu_bench.log; cat gpurun_out/sense_bench.log
