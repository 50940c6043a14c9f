mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rle.py tests/test_gpu_rle_dir.py tests/test_gpu_stress.py tests/test_gpu_baseline.py -x -q > gpurun_out/pytest_win.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_win.log
for rep in 1 2 3; do
  timeout 600 python bench.py --workload c4 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/k3w_base_$rep.log 2>&1
  for v in _variants/libbq_*.so; do
    n=$(basename $v .so)
    BQ_LIB=$PWD/$v timeout 600 python bench.py --workload c4 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/k3w_${n}_$rep.log 2>&1
  done
done
echo done
