mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --workload c4 > gpurun_out/bench_c4.log 2>&1; echo "bench c4 rc=$?" >> gpurun_out/bench_c4.log
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rle_count -s 3 -c 1 -o gpurun_out/prof_c4 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/ncu_c4.log 2>&1
echo done
