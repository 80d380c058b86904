# A/B of the CG loop: default build vs build/alt/*.so (+ tests with TESTS=1)
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 600 python -m pytest -q -x tests/test_gpu_sense_rank.py tests/test_gpu_sense.py tests/test_gpu_golden.py > gpurun_out/pdl_tests.log 2>&1; tail -2 gpurun_out/pdl_tests.log; fi
: > gpurun_out/pdl_sb.log
for rep in 1 2; do
for lib in paper_2202_14005_b200/libmdnn_b200.so build/alt/*.so; do
echo "== $lib" >> gpurun_out/pdl_sb.log
MDNN_B200_LIB=$lib timeout 300 python tools/sense_bench.py 320 368 15 8 512 512 32 4 --iters 20 >> gpurun_out/pdl_sb.log 2>&1
done
done
