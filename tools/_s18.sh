set -x
mkdir -p gpurun_out
python tools/zgemm_probe.py 3968 4000 128 8 10 0 >> gpurun_out/s18_probe.jsonl 2>&1
python tools/zgemm_probe.py 16128 16256 256 2 5 0 >> gpurun_out/s18_probe.jsonl 2>&1
python tools/zgemm_probe.py 8064 8128 256 4 5 0 >> gpurun_out/s18_probe.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_moments.py tests/test_gpu_solver.py -m gpu -q > gpurun_out/s18_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s18_tests.log
for c in 2 3 4; do python tools/cfg_twice.py $c 5 > gpurun_out/s18_cfg$c.log 2>&1; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 3 -c 1 -o gpurun_out/s18_zgemm_cfg2 -f python tools/zgemm_probe.py 3968 4000 128 8 2 0 > gpurun_out/s18_ncu_zgemm2.log 2>&1
