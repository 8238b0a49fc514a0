mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tail.py -x -q > gpurun_out/pytest_tail.log 2>&1; echo "rc $?" >> gpurun_out/pytest_tail.log
tail -n 4 gpurun_out/pytest_tail.log
for pn in reg smem; do echo "SSSVD_QR_PANEL=$pn"; SSSVD_QR_PANEL=$pn SSSVD_DEBUG=1 timeout 300 python tools/qr_time.py 2>&1 | grep thin_qr | awk 'NR%3==0'; done > gpurun_out/qr_time.log
cat gpurun_out/qr_time.log
