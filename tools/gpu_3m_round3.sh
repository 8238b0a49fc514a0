set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=6 > gpurun_out/3m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/3m_tests.log
python tools/zgemm_probe.py 16128 16256 256 2 5 0,2 > gpurun_out/3m_probe_final.jsonl 2>&1
python tools/zgemm_probe.py 3968 4000 128 8 10 0,2 >> gpurun_out/3m_probe_final.jsonl 2>&1
python bench.py --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/3m_bench5.jsonl 2> gpurun_out/3m_bench5.err
