mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pp_pytest.log 2>&1; echo "rc $?" >> gpurun_out/pp_pytest.log
tail -3 gpurun_out/pp_pytest.log
timeout 300 python tools/phase_ab.py 2 --reps 6 | cut -c1-250
SSSVD_PANEL_PREP=v1 timeout 300 python tools/phase_ab.py 2 --reps 6 | cut -c1-250
timeout 600 python tools/phase_ab.py 4 --reps 2 | cut -c1-250
