# one ncu --set full capture (one tool per gpurun call):  bash scripts/gpu_ncu.sh c2|c3|c4
mkdir -p gpurun_out
W=${1:-c2}
case $W in
  c2) K=count_kernel; S=6; C=2; P="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline";;
  c3) K=count_kernel; S=3; C=1; P="python bench.py --workload c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline";;
  c4) K=rle_sliced; S=3; C=1; P="python bench.py --workload c4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline";;
esac
$P > gpurun_out/plain_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$K -s $S -c $C -o gpurun_out/prof_$W $P > gpurun_out/ncu_$W.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$W.log
