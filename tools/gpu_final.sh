#!/bin/bash
# Round-end evidence pass: smoke, full GPU tests, every workload's bench line,
# the reference arm (C2), the ncu launch list and per-kernel DRAM traffic of
# the default bench, and one ncu --set full capture of the A^H A CG launch.
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for w in modl_c2 varnet_c3 modl_c5 sense_c4 modl_c1; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.log 2>&1; echo "bench rc=$?" >> $O/bench_$w.log
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference_c2.log 2>&1; echo "rc=$?" >> $O/bench_reference_c2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_modl_c2.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_list.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
   --log-file $O/traffic_modl_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_traffic.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_varnet_c3.csv \
   python bench.py --workload varnet_c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_list_vn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_normal_ws -s 10 -c 1 -o $O/prof_ahha_c2 -f \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_ahha.log 2>&1
tail -n 2 $O/smoke.log $O/pytest_gpu.log
for w in modl_c2 varnet_c3 modl_c5 sense_c4 modl_c1; do grep '^{' $O/bench_$w.log | tail -1 | cut -c1-200; done
