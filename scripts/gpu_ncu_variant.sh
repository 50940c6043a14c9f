# ncu --set full of the fresh-query kernels with a _variants/ library: V=<name> TAG=<suffix>
mkdir -p gpurun_out
export BQ_LIB=$PWD/_variants/libbq_$V.so
P="python bench.py --workload c4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_fresh.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KRE:-rle_count_wide_kernel|rle_resolve_kernel}" -s ${SKIP:-2} -c ${COUNT:-2} -o gpurun_out/prof_c4_fresh${TAG} $P > gpurun_out/ncu_fresh.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fresh.log
