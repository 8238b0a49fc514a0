set -x
mkdir -p gpurun_out
NCU="ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv"
SSSVD_LEAF=smem timeout 600 $NCU --log-file gpurun_out/s4_launches_cfg2_smem.csv python tools/profile_once.py 2 0 > gpurun_out/s4_ncu_smem.log 2>&1
SSSVD_LEAF_W=16 timeout 600 $NCU --log-file gpurun_out/s4_launches_cfg2_reg16.csv python tools/profile_once.py 2 0 > gpurun_out/s4_ncu_reg16.log 2>&1
timeout 600 $NCU --log-file gpurun_out/s4_launches_cfg2_reg32.csv python tools/profile_once.py 2 0 > gpurun_out/s4_ncu_reg32.log 2>&1
SSSVD_LEAF_W=8 timeout 600 $NCU --log-file gpurun_out/s4_launches_cfg2_reg8.csv python tools/profile_once.py 2 0 > gpurun_out/s4_ncu_reg8.log 2>&1
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_tail.py -m gpu -q > gpurun_out/s4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s4_tests.log
