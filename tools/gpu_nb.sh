mkdir -p gpurun_out
timeout 600 python tools/shard_sweep.py --config 2 --groups 4 2 --env "" "SSSVD_NB=256" 
timeout 900 python tools/shard_sweep.py --config 5 --sim 8:0 --groups 4 2 --env "" "SSSVD_NB=256"
timeout 900 python tools/shard_sweep.py --config 4 --groups 4 --env "" "SSSVD_NB=256"
