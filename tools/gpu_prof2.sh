#!/bin/bash
# ncu --set full captures of the RBF weight-gradient pass (VarNet C3) and the BN apply pass (MoDL C2)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rbf_wgrad_w -s 2 -c 1 \
   -o gpurun_out/prof_rbfw -f python bench.py --workload varnet_c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_rbfw.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_apply|k_thin_wgrad" -s 4 -c 3 \
   -o gpurun_out/prof_apply -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_apply.log 2>&1
tail -1 gpurun_out/ncu_rbfw.log gpurun_out/ncu_apply.log
