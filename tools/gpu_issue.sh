mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_solver.py -m gpu -x -q -k zgemm > gpurun_out/zi_pytest.log 2>&1; echo "rc $?" >> gpurun_out/zi_pytest.log
for s in 0 1 4; do for v in 0 8 9 10; do timeout 120 python tools/zgemm_variants.py --reps 10 --shape $s --variant $v; done; done > gpurun_out/zgemm_issue.jsonl 2>&1
for v in 0 8; do
  SSSVD_ZGEMM_V=$v timeout 400 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_zi$v.json 2> gpurun_out/bench_zi$v.err
done
tail -2 gpurun_out/zi_pytest.log; cat gpurun_out/zgemm_issue.jsonl | cut -c1-200
for v in 0 8; do python -c "import json,sys; d=json.load(open('gpurun_out/bench_zi$v.json')); print($v, d['value'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['phase_tflops'], d['step_ms'])"; done
