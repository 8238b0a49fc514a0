mkdir -p gpurun_out
SSSVD_DEBUG=1 timeout 600 python tools/cfg_twice.py 5 > gpurun_out/cfg5.log 2>&1; echo "cfg5 rc $?" >> gpurun_out/cfg5.log
SSSVD_DEBUG=1 timeout 600 python tools/cfg_twice.py 3 > gpurun_out/cfg3.log 2>&1; echo "cfg3 rc $?" >> gpurun_out/cfg3.log
grep -v "^\[sssvd\] \(jacobi_svd\|gram\)" gpurun_out/cfg5.log | tail -40; tail -4 gpurun_out/cfg3.log
