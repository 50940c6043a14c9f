# ncu --set full of the fresh-query RLE kernels on C4 (K3 rle_dir_kernel + K4 rle_count_kernel of the
# first full-size query; the warm-up query's two launches are skipped), plus the launch list
mkdir -p gpurun_out
P="python bench.py --workload c4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_fresh.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-rle_dir_kernel|rle_count_kernel|rle_resolve_kernel}" -s ${SKIP:-3} -c ${COUNT:-3} -o gpurun_out/prof_c4_fresh${TAG} $P > gpurun_out/ncu_fresh.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fresh.log
