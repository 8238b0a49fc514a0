# diagnostic gpurun call: config-5 GPU vs oracle with delta = 1e-12 on both sides (drops the
# roundoff-level directions of S that the reference default 1e-20 keeps)
mkdir -p gpurun_out
PARITY_DELTA=1e-12 timeout 2700 python tools/parity_full.py 5 0 > gpurun_out/parity5d.log 2>&1; echo "rc $?" >> gpurun_out/parity5d.log
tail -c 1500 gpurun_out/parity5d.log
