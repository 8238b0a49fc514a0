set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=6 > gpurun_out/3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/3m_tests.log
{
for d in 0 300 450 600 750 900 1200; do
  echo "# desync $d"
  SSSVD_ZGEMM_DESYNC=$d python tools/zgemm_probe.py 16128 16256 256 2 5 2,3
  SSSVD_ZGEMM_DESYNC=$d python tools/zgemm_probe.py 3968 4000 128 8 10 2,3
done
} > gpurun_out/3m_desync.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k regex:zgemm3m_kernel -s 1 -c 1 -o gpurun_out/3m4_zgemm_cfg5 -f python tools/zgemm_probe.py 16128 16256 256 2 2 3 > gpurun_out/3m4_ncu.log 2>&1
