mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_solver.py -m gpu -x -q -k zgemm > gpurun_out/zv0_pytest.log 2>&1; echo "rc $?" >> gpurun_out/zv0_pytest.log
for s in 0 1 2 4 5; do timeout 120 python tools/zgemm_variants.py --reps 10 --shape $s --variant 0; done > gpurun_out/zgemm_v0.jsonl 2>&1
timeout 400 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/bench_v0.json 2> gpurun_out/bench_v0.err
tail -2 gpurun_out/zv0_pytest.log; cat gpurun_out/zgemm_v0.jsonl | cut -c1-220
python -c "import json,sys; d=json.load(open('gpurun_out/bench_v0.json')); print(d['value'], d['e2e']['value'], d['roofline']['achieved'], d['roofline']['phase_tflops'], d['step_ms'])"
