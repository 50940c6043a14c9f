mkdir -p gpurun_out
for c in 0 64 128 256 1024; do
  echo "== chunk $c" >> gpurun_out/e2e.log
  timeout 600 python bench.py --no-cpu-baseline --steps 20 --e2e-steps 10 --e2e-chunk-mib $c >> gpurun_out/e2e.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_threshold.py -x -q -k sweep > gpurun_out/pytest_sweep.log 2>&1; echo rc=$? >> gpurun_out/pytest_sweep.log
