# one gpurun call: tests, smoke, bench lines, ncu launch list + one full capture
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-c2}; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?" >> gpurun_out/bench_$w.log
done
echo done
