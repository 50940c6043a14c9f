# library change check: RLE/directory/threshold tests, then the C4 A/B against _variants/
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rle.py tests/test_gpu_rle_dir.py tests/test_gpu_stress.py tests/test_gpu_sweep_stats.py tests/test_gpu_threshold.py tests/test_gpu_hygiene.py -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
bash scripts/gpu_ab.sh > /dev/null 2>&1
bash scripts/ab_report.sh > gpurun_out/ab_report.txt 2>&1
