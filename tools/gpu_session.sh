set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/test_gpu_solver.py -q -k "dgemm or zgemm" > gpurun_out/g3_gemm.log 2>&1; echo "rc=$?" >> gpurun_out/g3_gemm.log
python -m pytest tests/test_gpu_binding.py tests/test_gpu_moments.py -q > gpurun_out/g3_bind.log 2>&1; echo "rc=$?" >> gpurun_out/g3_bind.log
timeout 1200 python tools/parity_dump.py 1,2,3,4,5 > gpurun_out/g3_dump.log 2>&1; echo "rc=$?" >> gpurun_out/g3_dump.log
timeout 900 python tools/leaf_sweep.py 1,2 default SSSVD_ZGEMM=cpasync SSSVD_LEAF_W=8+SSSVD_LEAF_C=1 SSSVD_LEAF_W=8+SSSVD_LEAF_C=4 SSSVD_LEAF_W=16+SSSVD_LEAF_C=16 SSSVD_LEAF_W=8+SSSVD_LEAF_C=8 > gpurun_out/g3_sweep.log 2>&1
timeout 600 python tools/leaf_sweep.py 5 default SSSVD_ZGEMM=cpasync >> gpurun_out/g3_sweep.log 2>&1
