set -x
mkdir -p gpurun_out
python -m pytest tests/test_gpu_tail.py tests/test_gpu_pipeline.py -m gpu -q > gpurun_out/jac_tests.log 2>&1; echo "rc=$?" >> gpurun_out/jac_tests.log
SSSVD_JACOBI_PROF=1 SSSVD_TAIL_PROF=1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/jac_bench5.jsonl 2> gpurun_out/jac_prof.log
python -m pytest tests/test_gpu_parity_configs.py -m gpu -q -s > gpurun_out/jac_parity.log 2>&1; echo "rc=$?" >> gpurun_out/jac_parity.log
for c in 1 2 3 4; do python bench.py --config $c --steps 5 --no-cpu-baseline > gpurun_out/jac_bench_cfg$c.jsonl 2>/dev/null; done
