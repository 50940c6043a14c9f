# ncu --set full of K4s at T=20 on C4 streams (phase C heavy)
mkdir -p gpurun_out
python scripts/probe/c4_t_sweep.py 20 > gpurun_out/t20_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rle_sliced -s 4 -c 1 -o gpurun_out/prof_t20 python scripts/probe/c4_t_sweep.py 20 > gpurun_out/ncu_t20.log 2>&1
echo "rc=$?"
