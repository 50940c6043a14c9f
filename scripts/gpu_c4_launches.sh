# ncu launch list (durations) of the C4 bench's one-time kernels (directory, slice build) and queries
mkdir -p gpurun_out
P="python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_c4l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"rle_|slice_|Scan|arrange|sort_|iota|Radix" --log-file gpurun_out/launches_c4.csv $P > /dev/null 2>&1
echo "rc=$?"
