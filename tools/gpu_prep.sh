mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/prep_pytest.log 2>&1; echo "rc $?" >> gpurun_out/prep_pytest.log
tail -2 gpurun_out/prep_pytest.log
for i in 1 2; do
  timeout 300 python tools/phase_ab.py 2 --reps 6
  SSSVD_SPLIT_PREP=1 timeout 300 python tools/phase_ab.py 2 --reps 6
done 2>&1 | cut -c1-250
