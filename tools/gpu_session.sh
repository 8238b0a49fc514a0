set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/g1_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/g1_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g1_smoke.log
SSSVD_TAIL_PROF=1 timeout 300 python tools/cfg_twice.py 2 > gpurun_out/g1_cfg2.log 2>&1
SSSVD_TAIL_PROF=1 timeout 600 python tools/cfg_twice.py 5 > gpurun_out/g1_cfg5.log 2>&1
tail -3 gpurun_out/g1_tests.log gpurun_out/g1_smoke.log
