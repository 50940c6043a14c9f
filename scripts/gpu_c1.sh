mkdir -p gpurun_out
C="python bench.py --workload c1 --steps 20 --warmup 5"
$C > gpurun_out/c1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $C > /dev/null 2>&1
echo done
