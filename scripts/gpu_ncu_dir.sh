# ncu --set full of the K3a chain kernel on C4
mkdir -p gpurun_out
P="python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_c4d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rle_chain -c 1 -o gpurun_out/prof_dir $P > gpurun_out/ncu_dir.log 2>&1
echo "rc=$?"
