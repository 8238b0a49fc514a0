# diagnostic gpurun call: configs 1-4 GPU vs oracle with delta = 1e-12 on both sides
mkdir -p gpurun_out
for spec in "1 1" "2 0 1" "3 0" "4 1"; do
  PARITY_DELTA=1e-12 timeout 900 python tools/parity_full.py $spec >> gpurun_out/parity_delta.log 2>&1; echo "rc $? ($spec)" >> gpurun_out/parity_delta.log
done
grep "^rc" gpurun_out/parity_delta.log
