mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rle_dir.py tests/test_gpu_program.py tests/test_gpu_encode.py tests/test_gpu_rle.py -x -q > gpurun_out/pytest_q2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q2.log
timeout 600 python bench.py --workload frows --steps 20 > gpurun_out/bench_frows.log 2>&1; echo "rc=$?" >> gpurun_out/bench_frows.log
timeout 1200 python -m pytest tests/test_gpu_bench.py -x -q > gpurun_out/pytest_bench.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_bench.log
