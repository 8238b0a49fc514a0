mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tail.py -x -q > gpurun_out/pytest_tail.log 2>&1; echo "rc $?" >> gpurun_out/pytest_tail.log
tail -n 2 gpurun_out/pytest_tail.log
timeout 900 python tools/parity_full.py 1 1 > gpurun_out/parity1.log 2>&1
timeout 900 python tools/parity_full.py 2 0 1 > gpurun_out/parity2.log 2>&1
cat gpurun_out/parity1.log gpurun_out/parity2.log | tail -5
