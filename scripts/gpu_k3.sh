# the RLE directory (K3) and fresh-query path: smoke, RLE-related GPU tests, the C4
# bench line with the new K3 and (A/B) the previous two-kernel K3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_rle.py tests/test_gpu_baseline.py tests/test_gpu_hygiene.py tests/test_gpu_harness.py -x -q > gpurun_out/pytest_k3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k3.log
timeout 600 python bench.py --workload c4 --steps 10 --no-e2e > gpurun_out/bench_c4_new.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_new.log
BQ_RLE_K3=old timeout 600 python bench.py --workload c4 --steps 10 --no-e2e > gpurun_out/bench_c4_old.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4_old.log
echo done
