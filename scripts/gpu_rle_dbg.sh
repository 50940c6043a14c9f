mkdir -p gpurun_out
for d in 0 1 2; do BQ_RLE_DEBUG=$d timeout 900 python bench.py --workload c4 --steps 50 > gpurun_out/bench_c4_d$d.log 2>&1; done
echo done
