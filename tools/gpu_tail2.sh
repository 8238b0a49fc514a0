mkdir -p gpurun_out
SSSVD_DEBUG=1 SSSVD_TAIL_PROF=1 timeout 600 python tools/cfg_twice.py 2 > gpurun_out/tailprof_cfg2.log 2>&1; echo "rc $?" >> gpurun_out/tailprof_cfg2.log
tail -60 gpurun_out/tailprof_cfg2.log
