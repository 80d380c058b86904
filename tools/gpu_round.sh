#!/bin/bash
# Round-level GPU pass: smoke, full GPU tests, bench lines for every workload,
# launch list (ncu, gpu__time_duration) of the default bench.  Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_EXTRA} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-modl_c2}; do
  timeout 900 python bench.py --workload $w ${BENCH_ARGS} > gpurun_out/bench_$w.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$w.log
done
if [ -n "$NCU_LIST" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_list.log 2>&1
fi
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-modl_c2}; do grep '^{' gpurun_out/bench_$w.log | tail -1 | cut -c1-300; done
