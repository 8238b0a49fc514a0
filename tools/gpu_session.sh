set -x
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_configs.py > gpurun_out/g4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g4_tests.log
SSSVD_ZGEMM=tma python -m pytest tests/test_gpu_moments.py tests/test_gpu_pipeline.py -q > gpurun_out/g4_tma.log 2>&1; echo "rc=$?" >> gpurun_out/g4_tma.log
rm -rf gpurun_out/parity_dump
timeout 1200 python tools/parity_dump.py 1,2,3,4,5 > gpurun_out/g4_dump.log 2>&1; echo "rc=$?" >> gpurun_out/g4_dump.log
