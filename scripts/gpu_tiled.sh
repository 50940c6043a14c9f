# RLE parity tests + C4 bench (tile-major K4), then an ncu capture of the K4 launch.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rle.py -x -q > gpurun_out/pytest_tiled.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiled.log
timeout 900 python bench.py --workload c4 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_t2.log 2>&1 || exit 1
if [ -n "$PROF" ]; then
ncu --set full --clock-control none --import-source on -k regex:rle_tiled -s 3 -c 1 -o gpurun_out/prof_c4_rle_tiled python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
fi
echo done
