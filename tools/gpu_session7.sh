set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_solver.py -m gpu -q -x > gpurun_out/s7_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s7_tests.log
NCU="ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv"
SSSVD_LEAF_W=16 timeout 600 $NCU --log-file gpurun_out/s7_launches_cfg2_reg16.csv python tools/profile_once.py 2 0 > gpurun_out/s7_ncu_reg16.log 2>&1
timeout 600 $NCU --log-file gpurun_out/s7_launches_cfg2_reg32.csv python tools/profile_once.py 2 0 > gpurun_out/s7_ncu_reg32.log 2>&1
for c in 1 2 4; do
  python tools/cfg_twice.py $c > gpurun_out/s7_cfg${c}_reg.log 2>&1
done
SSSVD_LEAF_W=16 python tools/cfg_twice.py 2 > gpurun_out/s7_cfg2_reg_w16.log 2>&1
SSSVD_LEAF_W=8 python tools/cfg_twice.py 2 > gpurun_out/s7_cfg2_reg_w8.log 2>&1
SSSVD_LEAF_W=8 python tools/cfg_twice.py 4 > gpurun_out/s7_cfg4_reg_w8.log 2>&1
SSSVD_LEAF_W=16 python tools/cfg_twice.py 1 > gpurun_out/s7_cfg1_reg_w16.log 2>&1
SSSVD_LEAF_W=16 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:leaf_lu_reg_kernel -s 300 -c 1 -o gpurun_out/s7_leaf_reg16 -f python tools/profile_once.py 2 0 > gpurun_out/s7_ncu_leaf.log 2>&1
