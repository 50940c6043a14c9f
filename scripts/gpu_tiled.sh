# RLE parity tests + C4 bench (derived-layout K4 variants), optional ncu capture.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rle.py tests/test_serial.py -x -q > gpurun_out/pytest_tiled.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tiled.log
timeout 900 python bench.py --workload c4 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_sliced.log 2>&1 || exit 1
BQ_RLE_LAYOUT=tiled timeout 900 python bench.py --workload c4 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_tiled.log 2>&1
for d in 1 2; do BQ_RLE_DEBUG=$d timeout 900 python bench.py --workload c4 --steps 50 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_sliced_d$d.log 2>&1; done
if [ -n "$PROF" ]; then
ncu --set full --clock-control none --import-source on -k regex:$PROF -s 3 -c 1 -o gpurun_out/prof_c4_$PROF python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
fi
echo done
