mkdir -p gpurun_out
SSSVD_JACOBI_PROF=1 timeout 300 python tools/jacobi_time.py 512 1024 2048 > gpurun_out/jacobi_time2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tail.py -x -q > gpurun_out/pytest_tail2.log 2>&1; echo "tail rc $?" >> gpurun_out/pytest_tail2.log
cat gpurun_out/jacobi_time2.log; tail -3 gpurun_out/pytest_tail2.log
