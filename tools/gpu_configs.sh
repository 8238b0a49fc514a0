mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
for c in 1 2 3 4 5; do timeout 900 python tools/cfg_twice.py $c 2>&1 | grep call2; done > gpurun_out/configs.log
cat gpurun_out/configs.log
