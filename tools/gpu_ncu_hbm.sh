mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"assemble_kernel|moments_kernel|colnorm_partial" -c 4 -o gpurun_out/ncu_hbm python tools/one_solve.py 2 0 > gpurun_out/ncu_hbm.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"colnorm_partial" -c 3 -o gpurun_out/ncu_colnorm3 python tools/one_solve.py 3 0 > gpurun_out/ncu_hbm3.log 2>&1
echo "ncu rc $?" >> gpurun_out/ncu_hbm.log; tail -2 gpurun_out/ncu_hbm.log
