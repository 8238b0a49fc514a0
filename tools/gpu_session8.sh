set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=8 > gpurun_out/s8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s8_tests.log
python tools/zgemm_probe.py 3968 4000 128 8 10 0 >> gpurun_out/s8_probe.jsonl 2>&1
python tools/zgemm_probe.py 16128 16256 256 2 5 0 >> gpurun_out/s8_probe.jsonl 2>&1
SSSVD_ZGEMM_DESYNC=0 python tools/zgemm_probe.py 3968 4000 128 8 10 0 >> gpurun_out/s8_probe.jsonl 2>&1
SSSVD_ZGEMM_DESYNC=0 python tools/zgemm_probe.py 16128 16256 256 2 5 0 >> gpurun_out/s8_probe.jsonl 2>&1
python tools/cfg_twice.py 5 > gpurun_out/s8_cfg5_desync.log 2>&1
SSSVD_ZGEMM_DESYNC=0 python tools/cfg_twice.py 5 > gpurun_out/s8_cfg5_nodesync.log 2>&1
python tools/cfg_twice.py 2 > gpurun_out/s8_cfg2.log 2>&1
python tools/cfg_twice.py 4 > gpurun_out/s8_cfg4.log 2>&1
python tools/cfg_twice.py 3 > gpurun_out/s8_cfg3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 3 -c 1 -o gpurun_out/s8_zgemm_cfg5 -f python tools/zgemm_probe.py 16128 16256 256 2 2 0 > gpurun_out/s8_ncu_zgemm5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel -s 3 -c 1 -o gpurun_out/s8_zgemm_cfg2 -f python tools/zgemm_probe.py 3968 4000 128 8 2 0 > gpurun_out/s8_ncu_zgemm2.log 2>&1
