mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc $?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
timeout 600 python tools/shard_sweep.py --config 2 --groups 4 --env "" "SSSVD_ZGEMM=4m" "" "SSSVD_ZGEMM=4m"
timeout 900 python tools/shard_sweep.py --config 5 --sim 8:0 --groups 4 --env "" "SSSVD_ZGEMM=4m"
timeout 600 python tools/parity_full.py 1 1 2>&1 | tail -1
