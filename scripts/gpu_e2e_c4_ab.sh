mkdir -p gpurun_out
for rep in 1 2; do
timeout 900 python bench.py --workload c4 --steps 20 --no-cpu-baseline > gpurun_out/e2e_new_$rep.log 2>&1
BQ_LIB=$PWD/_variants/libbq_old.so timeout 900 python bench.py --workload c4 --steps 20 --no-cpu-baseline > gpurun_out/e2e_old_$rep.log 2>&1
done
