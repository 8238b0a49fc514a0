# GEMM warp-tile variants: isolated timing + bitwise check, then the bench under each variant
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_solver.py -m gpu -x -q -k zgemm > gpurun_out/zv_pytest.log 2>&1; echo "rc $?" >> gpurun_out/zv_pytest.log
timeout 600 python tools/zgemm_variants.py --reps 10 > gpurun_out/zgemm_variants.jsonl 2> gpurun_out/zgemm_variants.err
for v in 0 1 2 3; do
  SSSVD_ZGEMM_V=$v timeout 400 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_zv$v.json 2> gpurun_out/bench_zv$v.err
done
tail -2 gpurun_out/zv_pytest.log; cat gpurun_out/zgemm_variants.jsonl; tail -3 gpurun_out/zgemm_variants.err
for v in 0 1 2 3; do python -c "import json,sys; d=json.load(open('gpurun_out/bench_zv$v.json')); print($v, d['value'], d['roofline']['achieved'], d['roofline']['phase_tflops'], d['step_ms'])"; done
