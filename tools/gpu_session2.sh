set -x
mkdir -p gpurun_out
for d in 0 1000 2000 3000 4000 6000; do
  SSSVD_ZGEMM_DESYNC=$d python tools/zgemm_probe.py 3968 4000 128 8 10 0 >> gpurun_out/s2_probe.jsonl 2>&1
  SSSVD_ZGEMM_DESYNC=$d python tools/zgemm_probe.py 16128 16256 256 2 5 0 >> gpurun_out/s2_probe.jsonl 2>&1
done
python tools/zgemm_probe.py 3968 4000 128 8 10 1 >> gpurun_out/s2_probe.jsonl 2>&1
python tools/zgemm_probe.py 16128 16256 256 2 5 1 >> gpurun_out/s2_probe.jsonl 2>&1
for d in 0 2000 4000; do
  SSSVD_ZGEMM_DESYNC=$d python tools/cfg_twice.py 2 > gpurun_out/s2_cfg2_d$d.log 2>&1
  SSSVD_ZGEMM_DESYNC=$d python tools/cfg_twice.py 4 > gpurun_out/s2_cfg4_d$d.log 2>&1
done
python tools/cfg4_subspace.py 4 1e-12,1e-10,1e-8 > gpurun_out/s2_cfg4_subspace.jsonl 2> gpurun_out/s2_cfg4_subspace.err
python -m pytest tests/test_gpu_parity_configs.py -m gpu -q -k "fixture" > gpurun_out/s2_test_cfg5.log 2>&1
