# A/B of the tile-major RLE layout (BQ_RLE_TILED) on C4 plus the RLE parity tests.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rle.py -x -q > gpurun_out/pytest_tiled.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiled.log
for m in 2 0; do BQ_RLE_TILED=$m timeout 900 python bench.py --workload c4 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_t$m.log 2>&1; done
echo done
