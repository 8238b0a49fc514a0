mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tail.py -x -q > gpurun_out/pytest_tail.log 2>&1; echo "rc $?" >> gpurun_out/pytest_tail.log
tail -n 3 gpurun_out/pytest_tail.log
SSSVD_JACOBI_PROF=1 SSSVD_DEBUG=1 timeout 300 python tools/jacobi_time.py child 512 1024 2048 2>&1 | grep -v "jacobi_svd k"
