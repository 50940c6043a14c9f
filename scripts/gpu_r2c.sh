# round 2 checkpoint (second session): smoke, every GPU test, C4 + C2 bench lines, ncu of the fresh-query kernels
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in c4 c2; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?" >> gpurun_out/bench_$w.log
done
TAG=_r2e bash scripts/gpu_ncu_fresh.sh
