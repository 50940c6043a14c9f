# A/B of the C2 kernel: default libbq.so vs _variants/*.so, three interleaved 300-step runs each
mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 600 python bench.py --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/abc2_base_$rep.log 2>&1
  for v in _variants/libbq_*.so; do
    n=$(basename $v .so)
    BQ_LIB=$PWD/$v timeout 600 python bench.py --steps 300 --no-e2e --no-cpu-baseline > gpurun_out/abc2_${n}_$rep.log 2>&1
  done
done
echo done
