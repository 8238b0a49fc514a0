mkdir -p gpurun_out
SSSVD_DEBUG=1 SSSVD_TAIL_PROF=1 timeout 600 python tools/cfg_twice.py 2 > gpurun_out/tailprof_cfg2.log 2>&1; echo "rc $?" >> gpurun_out/tailprof_cfg2.log
SSSVD_JACOBI=grid SSSVD_DEBUG=1 SSSVD_TAIL_PROF=1 timeout 600 python tools/cfg_twice.py 2 > gpurun_out/tailprof_cfg2_grid.log 2>&1; echo "rc $?" >> gpurun_out/tailprof_cfg2_grid.log
SSSVD_DEBUG=1 SSSVD_TAIL_PROF=1 timeout 600 python tools/cfg_twice.py 5 > gpurun_out/tailprof_cfg5.log 2>&1; echo "rc $?" >> gpurun_out/tailprof_cfg5.log
grep "jacobi kernel\|call1" gpurun_out/tailprof_cfg2.log gpurun_out/tailprof_cfg2_grid.log
