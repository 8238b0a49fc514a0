mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_solver.py -m gpu -x -q -k zgemm > gpurun_out/zp2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/zp2_pytest.log
for s in 0 1 2 3 4 5; do for v in 0 1 6 7 8; do timeout 120 python tools/zgemm_variants.py --reps 10 --shape $s --variant $v; done; done > gpurun_out/zgemm_p2.jsonl 2>&1
for v in 0 6 7; do
  SSSVD_ZGEMM_V=$v timeout 400 python bench.py --steps 3 --no-cpu-baseline > gpurun_out/bench_zq$v.json 2> gpurun_out/bench_zq$v.err
done
tail -2 gpurun_out/zp2_pytest.log; cat gpurun_out/zgemm_p2.jsonl | cut -c1-220
for v in 0 6 7; do python -c "import json,sys; d=json.load(open('gpurun_out/bench_zq$v.json')); print($v, d['value'], d['roofline']['achieved'], d['roofline']['phase_tflops'], d['step_ms'])"; done
