# A/B of the default library and every _variants/ build on the C4 fresh-query line
mkdir -p gpurun_out
for rep in 1 2; do
  timeout 600 python bench.py --workload c4 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/abw_default_$rep.log 2>&1
  for v in _variants/libbq_*.so; do
    n=$(basename $v .so)
    BQ_LIB=$PWD/$v timeout 600 python bench.py --workload c4 --steps 30 --no-e2e --no-cpu-baseline > gpurun_out/abw_${n}_$rep.log 2>&1
  done
done
echo done
