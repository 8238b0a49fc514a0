set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=6 > gpurun_out/s10_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s10_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s10_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/s10_smoke.log
python bench.py > gpurun_out/s10_bench_cfg5.jsonl 2> gpurun_out/s10_bench_cfg5.err; echo "rc=$?" >> gpurun_out/s10_bench_cfg5.err
python bench.py --impl reference > gpurun_out/s10_ref_cfg5.jsonl 2> gpurun_out/s10_ref_cfg5.err
for c in 1 2 3 4; do
  python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/s10_bench_cfg$c.jsonl 2> gpurun_out/s10_bench_cfg$c.err
done
BENCH_PROFILER_RANGE=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/s10_launches_bench_cfg5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s10_ncu_bench5.log 2>&1; echo "rc=$?" >> gpurun_out/s10_ncu_bench5.log
