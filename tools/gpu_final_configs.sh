# one gpurun call: steady-state configs 1-5 (third call of each), config-1 full parity vs the
# oracle, config-5 8-GPU scaling estimate
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt
for c in 1 2 3 4 5; do timeout 900 python tools/cfg_twice.py $c 2>&1 | grep call2; done > gpurun_out/configs.log
timeout 900 python tools/parity_full.py 1 1 > gpurun_out/parity1.log 2>&1; echo "parity rc $?" >> gpurun_out/parity1.log
timeout 1500 python tools/scale_estimate.py --config 5 > gpurun_out/scale_cfg5.jsonl 2> gpurun_out/scale_cfg5.err; echo "scale rc $?" >> gpurun_out/scale_cfg5.err
cat gpurun_out/configs.log; tail -3 gpurun_out/parity1.log; cat gpurun_out/scale_cfg5.jsonl; tail -2 gpurun_out/scale_cfg5.err
