# persistent K3 check: directory / RLE tests under a short timeout (a look-back deadlock would hang), then C4 lines
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rle_dir.py -x -q > gpurun_out/pytest_k3p.log 2>&1; echo "dir rc=$?" >> gpurun_out/pytest_k3p.log
grep -q "dir rc=0" gpurun_out/pytest_k3p.log || exit 1
timeout 1200 python -m pytest tests/test_gpu_rle.py tests/test_gpu_stress.py tests/test_gpu_baseline.py tests/test_gpu_fullsize.py tests/test_gpu_sweep_stats.py tests/test_serial.py tests/test_gpu_hygiene.py -m gpu -x -q >> gpurun_out/pytest_k3p.log 2>&1; echo "rle rc=$?" >> gpurun_out/pytest_k3p.log
for r in 1 2; do
  timeout 600 python bench.py --workload c4 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/k3p_$r.log 2>&1
done
