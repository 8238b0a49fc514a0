set -x
mkdir -p gpurun_out
tools/lat_probe > gpurun_out/s11_lat.txt 2>&1
for v in 0 1; do
  SSSVD_LEAF_V=$v python tools/cfg_twice.py 2 > gpurun_out/s11_cfg2_v$v.log 2>&1
  SSSVD_LEAF_V=$v python tools/cfg_twice.py 1 > gpurun_out/s11_cfg1_v$v.log 2>&1
  SSSVD_LEAF_V=$v python tools/cfg_twice.py 4 > gpurun_out/s11_cfg4_v$v.log 2>&1
done
NCU="ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv"
SSSVD_LEAF_V=1 timeout 600 $NCU --log-file gpurun_out/s11_launches_cfg2_v1.csv python tools/profile_once.py 2 0 > gpurun_out/s11_ncu_v1.log 2>&1
SSSVD_LEAF_V=1 timeout 600 python -m pytest tests/test_gpu_moments.py tests/test_gpu_solver.py -m gpu -q -x > gpurun_out/s11_tests_v1.log 2>&1; echo "rc=$?" >> gpurun_out/s11_tests_v1.log
