# A/B of _variants/libbq_*.so on the C4 bench line and the C4 threshold sweep, three interleaved rounds
mkdir -p gpurun_out
for rep in 1 2 3; do
  for v in _variants/libbq_*.so; do
    n=$(basename $v .so)
    BQ_LIB=$PWD/$v timeout 900 python bench.py --workload c4 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/ab_c4_${n}_$rep.log 2>&1
  done
done
for v in _variants/libbq_*.so; do
  n=$(basename $v .so)
  BQ_LIB=$PWD/$v timeout 600 python scripts/probe/c4_t_sweep.py 10 20 30 > gpurun_out/abt_${n}.log 2>&1
done
echo done
