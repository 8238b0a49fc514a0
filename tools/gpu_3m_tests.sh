set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --durations=6 > gpurun_out/3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/3m_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/3m_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/3m_smoke.log
ncu --set full --clock-control none --import-source on -k regex:zgemm3m_kernel -s 3 -c 1 -o gpurun_out/3m_zgemm_cfg5 -f python tools/zgemm_probe.py 16128 16256 256 2 2 2 > gpurun_out/3m_ncu.log 2>&1
