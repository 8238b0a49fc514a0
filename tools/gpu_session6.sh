set -x
mkdir -p gpurun_out
SSSVD_LEAF_W=16 timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:leaf_lu_reg_kernel -s 300 -c 1 -o gpurun_out/s6_leaf_reg16 -f python tools/profile_once.py 2 0 > gpurun_out/s6_ncu_leaf.log 2>&1
SSSVD_LEAF=smem timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:leaf_lu_kernel -s 300 -c 1 -o gpurun_out/s6_leaf_smem16 -f python tools/profile_once.py 2 0 > gpurun_out/s6_ncu_leaf_smem.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 3 -c 1 -o gpurun_out/s6_zgemm_cfg5 -f python tools/zgemm_probe.py 16128 16256 256 2 2 0 > gpurun_out/s6_ncu_zgemm.log 2>&1
