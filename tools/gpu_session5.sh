set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_solver.py -m gpu -q > gpurun_out/s5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s5_tests.log
NCU="ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv"
SSSVD_LEAF_W=16 timeout 600 $NCU --log-file gpurun_out/s5_launches_cfg2_reg16.csv python tools/profile_once.py 2 0 > gpurun_out/s5_ncu_reg16.log 2>&1
for c in 1 2 4; do
  python tools/cfg_twice.py $c > gpurun_out/s5_cfg${c}_reg.log 2>&1
done
SSSVD_LEAF_W=16 python tools/cfg_twice.py 2 > gpurun_out/s5_cfg2_reg_w16.log 2>&1
SSSVD_LEAF_W=8 python tools/cfg_twice.py 2 > gpurun_out/s5_cfg2_reg_w8.log 2>&1
SSSVD_LEAF_W=8 python tools/cfg_twice.py 4 > gpurun_out/s5_cfg4_reg_w8.log 2>&1
SSSVD_LEAF_W=16 python tools/cfg_twice.py 1 > gpurun_out/s5_cfg1_reg_w16.log 2>&1
SSSVD_LEAF=smem python tools/cfg_twice.py 2 > gpurun_out/s5_cfg2_smem.log 2>&1
