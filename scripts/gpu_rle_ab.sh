mkdir -p gpurun_out
BQ_RLE_STAGED=0 timeout 1200 python -m pytest tests/test_gpu_rle.py -x -q > gpurun_out/pytest_rle0.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rle0.log
BQ_RLE_STAGED=1 timeout 1200 python -m pytest tests/test_gpu_rle.py -x -q > gpurun_out/pytest_rle1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_rle1.log
for m in 0 1; do BQ_RLE_STAGED=$m timeout 900 python bench.py --workload c4 --steps 50 > gpurun_out/bench_c4_m$m.log 2>&1; done
BQ_RLE_STAGED=0 timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/bench_c4_small.log 2>&1 && \
BQ_RLE_STAGED=0 ncu --set full --clock-control none --import-source on -k regex:rle_count -s 3 -c 1 -o gpurun_out/prof_c4_m0 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/ncu_c4.log 2>&1
echo done
