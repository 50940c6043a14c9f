# K3 variants: RLE GPU tests on the default library and every _variants/libbq_*.so,
# then the C4 fresh-query line for each (two interleaved rounds)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rle.py tests/test_gpu_baseline.py tests/test_gpu_hygiene.py tests/test_gpu_stress.py -x -q > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k3.log
for v in _variants/libbq_*.so; do
  n=$(basename $v .so)
  BQ_LIB=$PWD/$v timeout 900 python -m pytest tests/test_gpu_rle.py tests/test_gpu_stress.py -x -q > gpurun_out/pytest_$n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$n.log
done
for rep in 1 2; do
  timeout 600 python bench.py --workload c4 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/k3ab_base_$rep.log 2>&1
  for v in _variants/libbq_*.so; do
    n=$(basename $v .so)
    BQ_LIB=$PWD/$v timeout 600 python bench.py --workload c4 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/k3ab_${n}_$rep.log 2>&1
  done
done
echo done
