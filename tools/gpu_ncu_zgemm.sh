# cuBLAS comparator timing + one ncu --set full capture (source-level) of the trailing GEMM
mkdir -p gpurun_out
timeout 300 python tools/zgemm_variants.py --reps 10 --shape 0 > gpurun_out/zgemm_cmp.jsonl 2>&1
timeout 300 python tools/zgemm_variants.py --reps 10 --shape 4 >> gpurun_out/zgemm_cmp.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 1 -c 1 -o gpurun_out/ncu_zgemm_v0 python tools/zgemm_variants.py --reps 1 --shape 0 --variant 0 > gpurun_out/ncu_zgemm.log 2>&1
echo "ncu rc $?" >> gpurun_out/ncu_zgemm.log
cat gpurun_out/zgemm_cmp.jsonl; tail -3 gpurun_out/ncu_zgemm.log
