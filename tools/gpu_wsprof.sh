#!/bin/bash
# A^H A investigation pass: per-role clock64 timings (-DWS_PROF build in
# build/alt/libprof.so) and one ncu --set full capture (with source) of the
# ws CG launch at C2.
mkdir -p gpurun_out
MDNN_B200_LIB=build/alt/libprof.so timeout 300 python tools/sense_bench.py 320 368 15 8 --iters 2 > gpurun_out/wsprof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_normal_ws -s 12 -c 1 \
   -o gpurun_out/prof_ws -f python tools/sense_bench.py 320 368 15 8 --iters 4 > gpurun_out/ncu_ws.log 2>&1
tail -3 gpurun_out/ncu_ws.log; grep "ws cta" gpurun_out/wsprof.log | head -20
