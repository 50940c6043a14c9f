# quick C4 timing (+ optional RLE tests)
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then timeout 1200 python -m pytest tests/test_gpu_rle.py tests/test_serial.py -x -q > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log; fi
timeout 900 python bench.py --workload c4 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_q.log 2>&1
echo done
