# full measurement pass: every workload, the reference arm, and the ncu launch list of the default bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/box.txt 2>&1; nproc >> gpurun_out/box.txt
for w in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?" >> gpurun_out/bench_$w.log
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
P="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $P > /dev/null 2>&1
echo done
