# The evidence run of a round on one B200 (gpurun -- bash tools/gpu_session.sh): GPU tests, smoke, the bench
# line of every config, the reference arm, the scaling estimate, and the ncu launch list of the bench command
# (timed step only).
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -q --durations=6 > gpurun_out/ev_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ev_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ev_smoke.log
python bench.py > gpurun_out/ev_bench_cfg5.jsonl 2> gpurun_out/ev_bench_cfg5.err; echo "rc=$?" >> gpurun_out/ev_bench_cfg5.err
python bench.py --impl reference > gpurun_out/ev_ref_cfg5.jsonl 2> gpurun_out/ev_ref_cfg5.err
for c in 1 2 3 4; do
  python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/ev_bench_cfg$c.jsonl 2> gpurun_out/ev_bench_cfg$c.err
done
SSSVD_ZGEMM=4m python bench.py --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/ev_bench_cfg5_4m.jsonl 2> gpurun_out/ev_bench_cfg5_4m.err
python tools/scale_estimate.py --config 5 > gpurun_out/ev_scale_estimate_cfg5.jsonl 2> gpurun_out/ev_scale_estimate_cfg5.err
SSSVD_TAIL_PROF=1 python bench.py --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2> gpurun_out/ev_tail_prof_cfg5.err
python -m pytest tests/test_gpu_parity_configs.py -m gpu -q -s > gpurun_out/ev_parity_reports.log 2>&1; echo "rc=$?" >> gpurun_out/ev_parity_reports.log
BENCH_PROFILER_RANGE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/ev_launches_bench_cfg5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_bench5.log 2>&1; echo "rc=$?" >> gpurun_out/ev_ncu_bench5.log
