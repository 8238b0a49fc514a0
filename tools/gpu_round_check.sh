# one gpurun call: GPU tests, smoke, bench line, large-k Jacobi timings, config-5 tail breakdown
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/jacobi_time.py 1024 2048 > gpurun_out/jacobi_time.log 2>&1
timeout 600 python -m pytest tests/test_gpu_tail.py -x -q > gpurun_out/pytest_tail.log 2>&1; echo "tail rc $?" >> gpurun_out/pytest_tail.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
SSSVD_DEBUG=1 timeout 600 python tools/cfg_twice.py 5 > gpurun_out/cfg5.log 2>&1; echo "cfg5 rc $?" >> gpurun_out/cfg5.log
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; cat gpurun_out/jacobi_time.log gpurun_out/bench.json
