# round 2 checkpoint: smoke, every GPU test, the bench lines, then ncu (fresh-query kernels, full set)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for w in c2 c4 frows c1 c3; do
  timeout 900 python bench.py --workload $w > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?" >> gpurun_out/bench_$w.log
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
P="python bench.py --workload c4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline"
$P > gpurun_out/plain_fresh.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rle_dir_kernel|rle_count_kernel" -s 2 -c 2 -o gpurun_out/prof_c4_fresh $P > gpurun_out/ncu_fresh.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_fresh.log
echo done
