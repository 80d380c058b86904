#!/bin/bash
# Round-end refresh after the RBF changes: smoke, full GPU tests, VarNet C3 and MoDL C2
# bench lines, VarNet C3 launch list
mkdir -p gpurun_out/final2
O=gpurun_out/final2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for w in varnet_c3 modl_c2; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.log 2>&1; echo "bench rc=$?" >> $O/bench_$w.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_varnet_c3.csv \
   python bench.py --workload varnet_c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_list_vn.log 2>&1
tail -n 2 $O/smoke.log $O/pytest_gpu.log
for w in varnet_c3 modl_c2; do grep '^{' $O/bench_$w.log | tail -1 | cut -c1-200; done
