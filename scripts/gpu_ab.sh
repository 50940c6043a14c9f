# A/B: C4 timing of the default libbq.so and each _variants/libbq_*.so, interleaved twice.
mkdir -p gpurun_out
W=${WORKLOAD:-c4}
for rep in 1 2 3; do
  timeout 900 python bench.py --workload $W --steps 50 --no-e2e --no-cpu-baseline $AB_ARGS > gpurun_out/ab_${W}_base_$rep.log 2>&1
  for v in _variants/libbq_*.so; do
    n=$(basename $v .so)
    BQ_LIB=$PWD/$v timeout 900 python bench.py --workload $W --steps 50 --no-e2e --no-cpu-baseline $AB_ARGS > gpurun_out/ab_${W}_${n}_$rep.log 2>&1
  done
done
echo done
