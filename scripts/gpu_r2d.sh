# round 2 final checkpoint: smoke, every GPU test, all bench lines, launch list, ncu of the fresh-query kernels
bash scripts/gpu_full.sh
timeout 900 python bench.py --workload frows > gpurun_out/bench_frows.log 2>&1; echo "bench frows rc=$?" >> gpurun_out/bench_frows.log
TAG=_r2g bash scripts/gpu_ncu_fresh.sh
bash scripts/gpu_c4_launches.sh
