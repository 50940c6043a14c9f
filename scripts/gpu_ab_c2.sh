mkdir -p gpurun_out
for rep in 1 2; do
for v in base lb3; do
  case $v in base) L=paper_1402_4073_b200/libbq.so;; lb3) L=paper_1402_4073_b200/libbq_lb3.so;; esac
  for pad in 0 256 520; do
    echo "== $v pad=$pad" >> gpurun_out/ab_c2_$v.log
    BQ_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 300 --pad-words $pad >> gpurun_out/ab_c2_$v.log 2>&1
  done
done
done
echo done
