mkdir -p gpurun_out
for v in old new l2hint old new l2hint; do
  case $v in old) L=paper_1402_4073_b200/libbq_old.so;; new) L=paper_1402_4073_b200/libbq.so;; l2hint) L=paper_1402_4073_b200/libbq_l2hint.so;; esac
  BQ_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 300 >> gpurun_out/ab_c2_$v.log 2>&1
  BQ_LIB=$L timeout 600 python bench.py --workload c3 --steps 200 >> gpurun_out/ab_c3_$v.log 2>&1
done
echo done
