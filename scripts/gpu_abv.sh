# each _variants/ library: the RLE/directory tests under BQ_LIB; then the C4 A/B at T=50 (gpurun_out/t50)
# and, with AB_T10=1, at T=10 (gpurun_out/t10)
mkdir -p gpurun_out
for v in _variants/libbq_*.so; do
  n=$(basename $v .so)
  BQ_LIB=$PWD/$v timeout 900 python -m pytest tests/test_gpu_rle.py tests/test_gpu_rle_dir.py -x -q > gpurun_out/pytest_$n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$n.log
done
mkdir -p gpurun_out/t50; bash scripts/gpu_ab.sh > /dev/null 2>&1; mv gpurun_out/ab_c4_*.log gpurun_out/t50/ 2>/dev/null
if [ "$AB_T10" = "1" ]; then
  mkdir -p gpurun_out/t10; AB_ARGS="--c4-t 10" bash scripts/gpu_ab.sh > /dev/null 2>&1; mv gpurun_out/ab_c4_*.log gpurun_out/t10/ 2>/dev/null
fi
