# K4 change check: RLE tests (both K4 paths), full-size C4, then C4 A/B at T=50 and T=10
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rle.py tests/test_gpu_rle_dir.py tests/test_gpu_stress.py tests/test_gpu_sweep_stats.py tests/test_gpu_baseline.py -x -q > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k c4 > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full.log
mkdir -p gpurun_out/t50; bash scripts/gpu_ab.sh > /dev/null 2>&1; mv gpurun_out/ab_c4_*.log gpurun_out/t50/ 2>/dev/null
mkdir -p gpurun_out/t10; AB_ARGS="--c4-t 10" bash scripts/gpu_ab.sh > /dev/null 2>&1; mv gpurun_out/ab_c4_*.log gpurun_out/t10/ 2>/dev/null
