set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
python -m pytest tests -m gpu -q -s --durations=20 > gpurun_out/g2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g2_tests.log
timeout 2400 python tools/make_oracle_fixture.py 5 > gpurun_out/g2_fixture5.log 2>&1; echo "fixture rc=$?" >> gpurun_out/g2_fixture5.log
