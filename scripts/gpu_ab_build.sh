# ncu durations of the tile-sliced layout build kernels for each _variants/libbq_*.so on the C4 streams
mkdir -p gpurun_out
P="python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for v in _variants/libbq_*.so; do
  n=$(basename $v .so)
  BQ_LIB=$PWD/$v ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"slice_|sort_lit|arrange" --log-file gpurun_out/build_$n.csv $P > /dev/null 2>&1
done
echo done
