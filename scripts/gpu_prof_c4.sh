# ncu --set full of the C4 K4 launch (tile-major kernel by default; KERNEL=rle_count for the per-stream one)
mkdir -p gpurun_out
K=${KERNEL:-rle_tiled}
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_c4_$K python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
echo done
