# K3 iteration: RLE tests, the C4 fresh-query line, then one ncu --set full of rle_dir_kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rle.py tests/test_gpu_baseline.py tests/test_gpu_hygiene.py tests/test_gpu_stress.py -x -q > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k3.log
timeout 600 python bench.py --workload c4 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
P="python bench.py --workload c4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_k3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${K:-rle_dir_kernel}" -s 1 -c 1 -o gpurun_out/prof_k3 $P > gpurun_out/ncu_k3.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k3.log
