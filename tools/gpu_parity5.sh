# one gpurun call: full-size config-5 GPU vs CPU-oracle parity (the oracle factors the 64
# shifts of n = 16384 on the host cores: ~20 min), written to gpurun_out/parity_cfg5_mode0.json
mkdir -p gpurun_out
(nproc; free -g; lscpu | grep "Model name") > gpurun_out/host5.txt
timeout 3000 python tools/parity_full.py 5 0 > gpurun_out/parity5.log 2>&1; echo "parity5 rc $?" >> gpurun_out/parity5.log
cat gpurun_out/host5.txt; tail -3 gpurun_out/parity5.log
