mkdir -p gpurun_out
timeout 1500 python tools/shard_sweep.py --config 2 --groups 4 --env "" "SSSVD_LEAF_C=4" "SSSVD_LEAF_C=16" "SSSVD_LEAF_W=32,SSSVD_LEAF_C=8" "SSSVD_LEAF_W=32,SSSVD_LEAF_C=16" "SSSVD_LEAF_W=8,SSSVD_LEAF_C=8" "SSSVD_LEAF_W=8,SSSVD_LEAF_C=4" > gpurun_out/leaf_sweep.log 2>&1
cat gpurun_out/leaf_sweep.log
