set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=6 > gpurun_out/head_tests.log 2>&1; echo "rc=$?" >> gpurun_out/head_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/head_smoke.log
python bench.py > gpurun_out/head_bench_cfg5.jsonl 2> gpurun_out/head_bench_cfg5.err; echo "rc=$?" >> gpurun_out/head_bench_cfg5.err
python bench.py --config 1 --steps 20 --no-cpu-baseline > gpurun_out/head_bench_cfg1.jsonl 2>/dev/null
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active,power.draw,temperature.gpu --format=csv > gpurun_out/head_smi.log 2>&1
