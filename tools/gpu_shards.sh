mkdir -p gpurun_out
{
timeout 600 python tools/shard_sweep.py --config 5 --sim 8:0 --groups 1 2 4 8
timeout 600 python tools/shard_sweep.py --config 5 --sim 4:0 --groups 2 4 8
timeout 300 python tools/shard_sweep.py --config 2 --groups 2 4 8
timeout 300 python tools/shard_sweep.py --config 2 --sim 8:0 --groups 1 2
} > gpurun_out/shards.log 2>&1
cat gpurun_out/shards.log
