mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -c 7 -o gpurun_out/ncu_zgemm_cublas python tools/zgemm_variants.py --reps 1 --shape 0 --variant 6 > gpurun_out/ncu_cublas.log 2>&1
echo "rc $?" >> gpurun_out/ncu_cublas.log; tail -2 gpurun_out/ncu_cublas.log
