# per-kernel ncu durations of the C4 build kernels for the default lib and each variant (one ncu tool per call)
mkdir -p gpurun_out
P="python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_ab.log 2>&1 || exit 1
for v in "" _variants/libbq_*.so; do
  n=$( [ -z "$v" ] && echo base || basename $v .so )
  if [ -z "$v" ]; then
    ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"${K:-slice_|rle_chain|rle_dirfill}" --log-file gpurun_out/abl_$n.csv $P > /dev/null 2>&1
  else
    BQ_LIB=$PWD/$v ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"${K:-slice_|rle_chain|rle_dirfill}" --log-file gpurun_out/abl_$n.csv $P > /dev/null 2>&1
  fi
done
echo done
