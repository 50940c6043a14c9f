mkdir -p gpurun_out
for rep in 1 2; do
for v in nopdl pdl; do
  case $v in nopdl) L=paper_1402_4073_b200/libbq_nopdl.so;; pdl) L=paper_1402_4073_b200/libbq.so;; esac
  echo "== $v" >> gpurun_out/ab_pdl.log
  BQ_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 300 >> gpurun_out/ab_pdl.log 2>&1
  BQ_LIB=$L timeout 600 python bench.py --workload c3 --steps 200 >> gpurun_out/ab_pdl.log 2>&1
done
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
