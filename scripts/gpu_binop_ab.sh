# binop unroll variants on the (f)-rows line, the host CPU model, and the C4 line (host-overhead check)
mkdir -p gpurun_out
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt; free -g >> gpurun_out/lscpu.txt
timeout 900 python -m pytest tests/test_gpu_rle.py tests/test_gpu_hygiene.py -x -q > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k3.log
timeout 600 python bench.py --workload c4 --steps 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
for rep in 1 2; do
  timeout 600 python bench.py --workload frows --steps 20 > gpurun_out/ab_frows_base_$rep.log 2>&1
  for v in _variants/libbq_*.so; do
    n=$(basename $v .so)
    BQ_LIB=$PWD/$v timeout 600 python bench.py --workload frows --steps 20 > gpurun_out/ab_frows_${n}_$rep.log 2>&1
  done
done
echo done
