set -x
mkdir -p gpurun_out
python tools/zgemm_probe.py 16128 16256 256 2 5 0,2 > gpurun_out/fin_probe.jsonl 2>&1
python tools/zgemm_probe.py 3968 4000 128 8 10 0,2 >> gpurun_out/fin_probe.jsonl 2>&1
python -m pytest tests -m gpu -q --durations=6 > gpurun_out/fin_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fin_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin_smoke.log
python bench.py > gpurun_out/fin_bench_cfg5.jsonl 2> gpurun_out/fin_bench_cfg5.err; echo "rc=$?" >> gpurun_out/fin_bench_cfg5.err
for c in 1 2 3 4; do
  python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/fin_bench_cfg$c.jsonl 2> gpurun_out/fin_bench_cfg$c.err
done
