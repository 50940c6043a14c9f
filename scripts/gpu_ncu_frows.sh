mkdir -p gpurun_out
P="python scripts/frows_kernels.py"
$P > gpurun_out/plain_frows.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"binop_kernel|enc_|bq_prog" -o gpurun_out/prof_frows $P > gpurun_out/ncu_frows.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_frows.log
