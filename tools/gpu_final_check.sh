# last gpurun call of the round: GPU tests + smoke at HEAD, and one ncu --set full capture of the
# default trailing-update GEMM (shape 0 = config-2 block-0 update, default variant)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 300 python tools/zgemm_variants.py --reps 5 --shape 0 > gpurun_out/zgemm_plain.log 2>&1; echo "plain rc $?" >> gpurun_out/zgemm_plain.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 1 -c 1 -o gpurun_out/ncu_zgemm_final python tools/zgemm_variants.py --reps 1 --shape 0 --variant 0 > gpurun_out/ncu_zgemm.log 2>&1; echo "ncu rc $?" >> gpurun_out/ncu_zgemm.log
tail -n 2 gpurun_out/pytest_gpu.log; tail -n 2 gpurun_out/smoke.log; tail -n 4 gpurun_out/zgemm_plain.log; tail -n 1 gpurun_out/ncu_zgemm.log
