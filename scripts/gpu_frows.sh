mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rle.py tests/test_gpu_encode.py tests/test_gpu_program.py -x -q > gpurun_out/pytest_enc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_enc.log
timeout 900 python bench.py --workload frows --steps 20 > gpurun_out/bench_frows.log 2>&1; echo "rc=$?" >> gpurun_out/bench_frows.log
