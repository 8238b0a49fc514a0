set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_solver.py tests/test_gpu_pipeline.py -m gpu -q -x > gpurun_out/s3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3_tests.log
for c in 1 2 4; do
  python tools/cfg_twice.py $c > gpurun_out/s3_cfg${c}_reg.log 2>&1
  SSSVD_LEAF=smem python tools/cfg_twice.py $c > gpurun_out/s3_cfg${c}_smem.log 2>&1
done
SSSVD_LEAF_W=16 python tools/cfg_twice.py 2 > gpurun_out/s3_cfg2_reg_w16.log 2>&1
SSSVD_LEAF_W=8 python tools/cfg_twice.py 4 > gpurun_out/s3_cfg4_reg_w8.log 2>&1
SSSVD_LEAF_W=16 python tools/cfg_twice.py 1 > gpurun_out/s3_cfg1_reg_w16.log 2>&1
python tools/cfg_twice.py 5 > gpurun_out/s3_cfg5_reg_desync.log 2>&1
SSSVD_ZGEMM_DESYNC=0 python tools/cfg_twice.py 5 > gpurun_out/s3_cfg5_reg_nodesync.log 2>&1
SSSVD_LEAF=smem SSSVD_ZGEMM_DESYNC=0 python tools/cfg_twice.py 5 > gpurun_out/s3_cfg5_smem_nodesync.log 2>&1
python tools/cfg4_subspace.py 4 1e-12,1e-10,1e-9,1e-8 > gpurun_out/s3_cfg4_subspace.jsonl 2> gpurun_out/s3_cfg4_subspace.err
timeout 900 python -m pytest tests/test_gpu_parity_configs.py -m gpu -q -x -k "live_oracle" -s > gpurun_out/s3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/s3_parity.log
