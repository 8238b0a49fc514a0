mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
SSSVD_TAIL_PROF=1 timeout 600 python tools/cfg_twice.py 5 > gpurun_out/tailprof_cfg5.log 2>&1; echo "rc $?" >> gpurun_out/tailprof_cfg5.log
tail -n 5 gpurun_out/pytest_gpu.log; tail -n 26 gpurun_out/tailprof_cfg5.log
