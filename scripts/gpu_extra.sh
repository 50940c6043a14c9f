# the extra workloads at N=1 (c1 c3 c4 c5), quick
mkdir -p gpurun_out
for w in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --steps 30 > gpurun_out/extra_$w.log 2>&1; echo "rc=$?" >> gpurun_out/extra_$w.log
done
