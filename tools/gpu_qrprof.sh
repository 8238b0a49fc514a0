mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qr_launches.csv python tools/qr_launches.py 16384 2048 > gpurun_out/qr_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/qr_launches.csv > gpurun_out/qr_launch_summary.txt 2>&1
SSSVD_DEBUG=1 SSSVD_TAIL_PROF=1 timeout 600 python tools/cfg_twice.py 5 > gpurun_out/tailprof_cfg5.log 2>&1; echo "rc $?" >> gpurun_out/tailprof_cfg5.log
cat gpurun_out/qr_launch_summary.txt; grep -v "jacobi_svd k\|gram " gpurun_out/tailprof_cfg5.log | tail -28
