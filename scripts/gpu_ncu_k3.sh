# ncu --set full of the fresh-query K3 (rle_dir_kernel) on C4, after the RLE tests pass
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rle.py tests/test_gpu_baseline.py tests/test_gpu_hygiene.py tests/test_gpu_stress.py -x -q > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k3.log
P="python bench.py --workload c4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_k3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rle_dir_kernel" -s 1 -c 1 -o gpurun_out/prof_k3 $P > gpurun_out/ncu_k3.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_k3.log
