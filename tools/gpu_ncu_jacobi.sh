mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_grid_block -c 1 -o gpurun_out/ncu_jacobi_grid python tools/jacobi_time.py child 2048 > gpurun_out/ncu_jacobi.log 2>&1
echo "ncu rc $?" >> gpurun_out/ncu_jacobi.log
tail -3 gpurun_out/ncu_jacobi.log
SSSVD_TAIL_PROF=1 timeout 600 python tools/cfg_twice.py 2 > gpurun_out/tailprof_cfg2.log 2>&1
tail -n 20 gpurun_out/tailprof_cfg2.log
