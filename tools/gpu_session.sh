set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/s1_gpu.txt
python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/s1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s1_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s1_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s1_smoke.log
python bench.py > gpurun_out/s1_bench_cfg5.jsonl 2> gpurun_out/s1_bench_cfg5.err; echo "rc=$?" >> gpurun_out/s1_bench_cfg5.err
python bench.py --config 2 --steps 10 > gpurun_out/s1_bench_cfg2.jsonl 2> gpurun_out/s1_bench_cfg2.err
python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/s1_bench_cfg1.jsonl 2> gpurun_out/s1_bench_cfg1.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/s1_ref_cfg5.jsonl 2> gpurun_out/s1_ref_cfg5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s1_launches_cfg2.csv python tools/profile_once.py 2 0 > gpurun_out/s1_ncu_cfg2.log 2>&1
