set -x
mkdir -p gpurun_out
python bench.py --config 3 --steps 6 --no-cpu-baseline > gpurun_out/s15_bench_cfg3.jsonl 2> gpurun_out/s15_bench_cfg3.err
python bench.py --config 2 --steps 10 --no-cpu-baseline > gpurun_out/s15_bench_cfg2.jsonl 2> gpurun_out/s15_bench_cfg2.err
python bench.py --config 4 --steps 5 --no-cpu-baseline > gpurun_out/s15_bench_cfg4.jsonl 2> gpurun_out/s15_bench_cfg4.err
python bench.py --config 1 --steps 10 --no-cpu-baseline > gpurun_out/s15_bench_cfg1.jsonl 2> gpurun_out/s15_bench_cfg1.err
python bench.py --no-cpu-baseline > gpurun_out/s15_bench_cfg5.jsonl 2> gpurun_out/s15_bench_cfg5.err
