# K4 check: RLE parity tests, then the C4 fresh-query line at T = 50 (twice), 10 and 20
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_rle.py tests/test_gpu_baseline.py tests/test_gpu_fullsize.py tests/test_gpu_stress.py tests/test_gpu_hypothesis.py -m gpu -x -q > gpurun_out/pytest_k4w.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k4w.log
for r in 1 2; do
  timeout 600 python bench.py --workload c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_$r.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_$r.log
done
for t in 10 20; do
  timeout 600 python bench.py --workload c4 --c4-t $t --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_t${t}.log 2>&1
done
