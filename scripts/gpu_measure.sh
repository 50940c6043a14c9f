# full measurement pass: every workload, then ncu evidence for the top kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/box.txt 2>&1; nproc >> gpurun_out/box.txt
for w in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?" >> gpurun_out/bench_$w.log
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
# ncu: launch list of the default bench, and one full capture per top kernel
P="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $P > /dev/null 2>&1
$P > gpurun_out/plain_c2b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:count_kernel -s 6 -c 2 -o gpurun_out/prof_c2 $P > /dev/null 2>&1
Q="python bench.py --workload c3 --steps 3 --warmup 3"
$Q > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:count_kernel -s 3 -c 1 -o gpurun_out/prof_c3 $Q > /dev/null 2>&1
R="python bench.py --workload c4 --steps 3 --warmup 3"
$R > gpurun_out/plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rle_count -s 3 -c 1 -o gpurun_out/prof_c4 $R > /dev/null 2>&1
echo done
