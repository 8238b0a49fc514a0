mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_moments.py -m gpu -x -q > gpurun_out/trsm_pytest.log 2>&1; echo "rc $?" >> gpurun_out/trsm_pytest.log
tail -2 gpurun_out/trsm_pytest.log
SSSVD_DEBUG_PHASE=1 timeout 300 python tools/phase_ab.py 2 --reps 10 > gpurun_out/outl.log 2>&1
grep -c "graph device" gpurun_out/outl.log; grep "graph device" gpurun_out/outl.log | awk '{print $5, $9}' | tr '\n' ' '; echo; grep phase_ms gpurun_out/outl.log | cut -c1-250
SSSVD_TRSM=warp timeout 300 python tools/phase_ab.py 2 --reps 6 | cut -c1-250
timeout 300 python tools/phase_ab.py 2 --reps 6 | cut -c1-250
