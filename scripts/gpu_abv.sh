# each _variants/ library: the RLE/directory tests under BQ_LIB, then the C4 A/B
mkdir -p gpurun_out
for v in _variants/libbq_*.so; do
  n=$(basename $v .so)
  BQ_LIB=$PWD/$v timeout 900 python -m pytest tests/test_gpu_rle.py tests/test_gpu_rle_dir.py -x -q > gpurun_out/pytest_$n.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$n.log
done
bash scripts/gpu_ab.sh > /dev/null 2>&1
