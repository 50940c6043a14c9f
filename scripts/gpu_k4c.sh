# K4c check: RLE parity tests, then the C4 fresh-query line at T = 50, 10, 20, 30
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_rle.py tests/test_gpu_baseline.py tests/test_gpu_fullsize.py tests/test_gpu_stress.py tests/test_gpu_hypothesis.py -m gpu -x -q > gpurun_out/pytest_k4c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k4c.log
timeout 600 python bench.py --workload c4 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/k4c_t50.log 2>&1
for t in 10 20 30; do
  timeout 600 python bench.py --workload c4 --c4-t $t --no-e2e --no-cpu-baseline > gpurun_out/k4c_t${t}.log 2>&1
done
